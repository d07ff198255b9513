"""Summarise ncu captures (gpurun_out/) into a committed text file under profiles/.

    python scripts/ncu_summary.py ROUND_TAG [gpurun_out]

Reads gpurun_out/launches.csv (the `--metrics gpu__time_duration.sum
--clock-control none` launch list of a bench run) and every
gpurun_out/prof_*.ncu-rep (`--set full` captures), and writes
profiles/<tag>_ncu_summary.txt: the per-kernel launch list with each kernel's
share of the step, then per captured kernel the duration, DRAM bytes
(the roofline `traffic`), throughputs, occupancy, issue efficiency, top
stall reasons and shared-memory wavefronts.
"""
import csv
import glob
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                unit = d.get("Metric Unit", "ns")
                ns = v * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(unit, 1)
                out.append((d["Kernel Name"], ns))
    return out


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    if len(rows) < 3:
        return {}, {}
    h, units, v = rows[0], rows[1], rows[2]
    return dict(zip(h, v)), dict(zip(h, units))


def main():
    tag = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    lines = [f"# ncu summary {tag} (source: {src}; clock-control none; cold-cache serialised launches)", ""]
    lp = os.path.join(src, "launches.csv")
    if os.path.exists(lp):
        ls = launches(lp)
        tot = defaultdict(float)
        cnt = defaultdict(int)
        for k, ns in ls:
            name = k.split("(")[0]
            tot[name] += ns
            cnt[name] += 1
        ours = {k: v for k, v in tot.items() if "uzip::" in k}
        step = sum(ours.values())
        lines.append("## launch list (uzip kernels; share of the uzip step)")
        for k, v in sorted(ours.items(), key=lambda kv: -kv[1]):
            lines.append(f"{k:40s} launches={cnt[k]:4d} mean={v / cnt[k] / 1e3:10.2f} us share={v / step:6.3f}")
        lines.append("")
    traffic = {}
    for rep in sorted(glob.glob(os.path.join(src, "prof_*.ncu-rep"))):
        v, u = raw(rep)
        if not v:
            continue
        try:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tb = sum(float(v[k].replace(",", "")) * scale.get(u.get(k, "byte"), 1)
                     for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            traffic[v.get("Kernel Name", rep).split("(")[0]] = int(tb)
        except (KeyError, ValueError):
            pass
        lines.append(f"## {os.path.basename(rep)}: {v.get('Kernel Name', '')[:90]}")
        for k in KEYS:
            if k in v:
                lines.append(f"  {k:75s} {v[k]:>16s} {u.get(k, '')}")
        stalls = []
        for k, x in v.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(x), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        lines.append("  top stalls (warps per issue): " +
                     ", ".join(f"{n}={x:.2f}" for x, n in sorted(stalls, reverse=True)[:6]))
        lines.append("")
    import json
    json.dump(traffic, open(os.path.join(ROOT, "profiles", f"{tag}_traffic.json"), "w"), indent=1)
    out = os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.txt")
    open(out, "w").write("\n".join(lines) + "\n")
    print(out)


if __name__ == "__main__":
    main()
