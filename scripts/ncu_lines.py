"""Attribute an ncu SASS source page (instructions executed, stall samples) to CUDA source lines.

    python scripts/ncu_lines.py LIB.so KERNEL_MANGLED_SUBSTR sass_page.csv [top]

LIB.so is the library the capture ran (built with -lineinfo); the SASS page is
`ncu -i REP --page source --csv --print-source sass`.  Prints the top source
lines by executed warp instructions and by stall samples.
"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict


def line_map(lib, kern):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
    for f in sorted(os.listdir(d)):
        if not f.endswith(".cubin"):
            continue
        dis = subprocess.run(["nvdisasm", "-g", os.path.join(d, f)], capture_output=True, text=True).stdout
        start = dis.find(f"\n{kern}")
        if start < 0:
            # substring match on a function label
            m = re.search(r"\n(_Z\S*" + re.escape(kern) + r"\S*):\n", dis)
            if not m:
                continue
            start = m.start()
        nxt = [e for e in (dis.find("\n.nv.", start + 10), dis.find("\n.text.", dis.find("\n.text.", start) + 5))
               if e > 0]
        end = min(nxt) if nxt else -1  # the next section: addresses restart per function
        body = dis[start:end if end > 0 else None]
        amap, cur = {}, "?"
        for ln in body.splitlines():
            m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if m:
                amap[int(m.group(1), 16)] = cur
        return amap
    raise SystemExit(f"kernel {kern} not found in {lib}")


def main():
    lib, kern, page = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    amap = line_map(lib, kern)
    rows = list(csv.reader(open(page)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    i_addr, i_inst, i_samp = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index(
        "Warp Stall Sampling (All Samples)")
    inst, samp = defaultdict(float), defaultdict(float)
    tot_i = tot_s = 0.0
    base = None
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= i_samp or not r[i_addr].startswith("0x"):
            continue
        a = int(r[i_addr], 16)
        base = a if base is None else base  # the page lists absolute addresses from the kernel's start
        a -= base
        key = amap.get(a, "?")
        v, s = float(r[i_inst] or 0), float(r[i_samp] or 0)
        inst[key] += v
        samp[key] += s
        tot_i += v
        tot_s += s
    print(f"total warp instructions {tot_i:.0f}, stall samples {tot_s:.0f}")
    print(f"{'line':28s} {'inst':>12s} {'%inst':>6s} {'%samp':>6s}")
    for k in sorted(inst, key=lambda k: -inst[k])[:top]:
        print(f"{k:28s} {inst[k]:12.0f} {100 * inst[k] / tot_i:6.2f} {100 * samp[k] / max(1, tot_s):6.2f}")


if __name__ == "__main__":
    main()
