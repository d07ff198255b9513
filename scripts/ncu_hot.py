"""Per-source-line stall samples and instructions of one kernel from an ncu SASS source page.

    python scripts/ncu_hot.py LIB.so KERNEL_MANGLED_SUBSTR sass_page.csv [top]

Like ncu_lines.py but sorted by stall samples, with the two hottest SASS instructions of each line.
"""
import csv
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_lines as nl  # noqa: E402


def main():
    lib, kern, page = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    amap = nl.line_map(lib, kern)
    rows = list(csv.reader(open(page)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    ia, isamp, ins = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    samp, inst, src = defaultdict(float), defaultdict(float), defaultdict(list)
    base, ts, ti = None, 0.0, 0.0
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= isamp or not r[ia].startswith("0x"):
            continue
        a = int(r[ia], 16)
        base = a if base is None else base
        k = amap.get(a - base, "?")
        s, i = float(r[isamp] or 0), float(r[ins] or 0)
        samp[k] += s
        inst[k] += i
        ts += s
        ti += i
        src[k].append((s, r[1].strip()))
    print(f"total warp instructions {ti:.0f}, stall samples {ts:.0f}")
    for k in sorted(samp, key=lambda k: -samp[k])[:top]:
        hot = sorted(src[k], reverse=True)[:2]
        print(f"{k:28s} %samp {100 * samp[k] / ts:6.2f}  %inst {100 * inst[k] / ti:6.2f}  {hot}")


if __name__ == "__main__":
    main()
