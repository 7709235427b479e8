"""Per-kernel SASS instruction-class counts of the built objects (cuobjdump),
proving which kernels run on tcgen05 / TMEM / TMA (bulk copy) hardware.

usage: python profiles/sass_counts.py > profiles/sass_counts_r2.json
Mnemonics (B200_PROFILING.md): UTCHMMA / UTCQMMA = tcgen05.mma, UTCBAR =
tcgen05.commit, LDTM = tcgen05.ld, UBLKCP = cp.async.bulk (TMA bulk copy),
UBLKPF = cp.async.bulk.prefetch.L2, SYNCS = mbarrier ops, FFMA / HFMA2 =
CUDA-core math, LDG = ordinary global loads.
"""
import json
import os
import re
import subprocess

OBJ = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2603_09983_b200", "_lib", "obj")
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "UBLKCP", "UBLKPF", "UTMALDG", "SYNCS", "FFMA", "HFMA2", "LDG", "STG",
        "SHFL", "MUFU"]


def main():
    out = {}
    for f in sorted(os.listdir(OBJ)):
        if not f.endswith(".cu.o"):
            continue
        sass = subprocess.run(["cuobjdump", "-sass", os.path.join(OBJ, f)], capture_output=True, text=True).stdout
        fn = None
        for line in sass.splitlines():
            m = re.match(r"\s+Function : (\S+)", line)
            if m:
                fn = m.group(1)
                out.setdefault(f, {})[fn] = {k: 0 for k in KEYS}
                continue
            m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
            if fn and m:
                op = m.group(1)
                for k in KEYS:
                    if op == k:
                        out[f][fn][k] += 1
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
