"""Extract the hot loops of the uzip kernels from cuobjdump SASS (no GPU needed).

    python scripts/sass_extract.py ROUND_TAG

For each listed kernel it writes the instruction-mix histogram of the whole
function and the densest VOTE-containing window (the rANS round loop) to
profiles/<tag>_sass_<kernel>.txt, so the committed listing shows what the
rounds compile to (LDS/VOTE/POPC/IMAD.HI ... and the absence of local memory).
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2604_17172_b200", "libuzip.so")
KERNELS = {
    "k_fused_bf16_b4096_encode": "_ZN4uzip7k_fusedILi0ELi4096ELb0ELi3ELb0EEEvNS_4PlanE",
    "k_fused_bf16_b4096_decode": "_ZN4uzip7k_fusedILi0ELi4096ELb0ELi4ELb1EEEvNS_4PlanE",
    "k_fused_bf16_b4096_reduce": "_ZN4uzip7k_fusedILi0ELi4096ELb1ELi3ELb0EEEvNS_4PlanE",
    "k_decode_bf16": "_ZN4uzip8k_decodeILi0EEEvPKhmPhmNS_7CodecWsEPi",
    "k_hist_bf16": "_ZN4uzip6k_histILi0EEEvNS_4PlanE",
}


def sass(fn):
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, LIB], capture_output=True, text=True).stdout
    lines = []
    for l in out.splitlines():
        m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(.*?);", l)
        if m:
            lines.append((m.group(1), m.group(2).strip()))
    return lines


def main():
    tag = sys.argv[1]
    for name, fn in KERNELS.items():
        ins = sass(fn)
        if not ins:
            continue
        ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for _, t in ins)
        # the fast-path rounds: VOTEs outside the compiler's divergent fallback (WARPSYNC.COLLECTIVE) blocks
        # (encode variant: the encoder's rounds, marked by IMAD.HI -- the reciprocal division -- next
        # to each VOTE; otherwise the decoder's rounds would be picked from the same kernel)
        enc = name.endswith("_encode")
        votes = [i for i, (_, t) in enumerate(ins) if "VOTE.ANY R" in t
                 and "WARPSYNC.COLLECTIVE" not in ins[i - 1][1]
                 and (not enc or any("IMAD.HI" in u for _, u in ins[max(0, i - 16): i + 16]))]
        best, lo = 0, 0
        nv = 4 if enc else 12  # the encoder's loop body is one group of UZIP_ENC_GROUP = 4 rounds
        for i in range(len(votes)):  # densest window of nv consecutive VOTEs
            j = min(len(votes) - 1, i + nv - 1)
            span = votes[j] - votes[i]
            if j - i == nv - 1 and (best == 0 or span < best):
                best, lo = span, votes[i]
        with open(os.path.join(ROOT, "profiles", f"{tag}_sass_{name}.txt"), "w") as f:
            f.write(f"# {name}: {fn}\n# {len(ins)} SASS instructions; cuobjdump -sass of libuzip.so (sm_100a)\n")
            f.write("# local-memory ops (spills): %d\n" % sum(v for k, v in ops.items() if k.startswith(("LDL", "STL"))))
            f.write("# instruction mix (top 30): " + ", ".join(f"{k}={v}" for k, v in ops.most_common(30)) + "\n\n")
            if votes:
                f.write("# hot loop window (%d rANS rounds around the densest VOTE run%s)\n"
                        % (nv, " of the encoder" if enc else ""))
                for a, t in ins[max(0, lo - 20): lo + best + 30]:
                    f.write(f"/*{a}*/ {t}\n")
        print(name, len(ins))


if __name__ == "__main__":
    main()
