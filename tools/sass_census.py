"""Per-kernel SASS opcode census of the built library (cuobjdump -sass), the
instruction-level evidence that the hot kernels use tcgen05 / TMA / TMEM:

  UTCHMMA / UTCQMMA  tcgen05.mma (tensor core, accumulator in TMEM)
  UTCBAR             tcgen05.commit (MMA completion -> mbarrier)
  STTM / LDTM        tcgen05.st / tcgen05.ld (registers <-> TMEM)
  UBLKCP             cp.async.bulk (TMA bulk copy engine)
  UTMALDG            cp.async.bulk.tensor (TMA tensor-map load)
  LDGSTS             cp.async (16-byte async global -> shared)
  FFMA / SHFL        SIMT FMA and warp shuffles

Usage: python tools/sass_census.py [lib.so] > profiles/r02_sass_census.txt
"""
import collections
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(HERE, "paper_1412_0680_b200", "_lib", "libstmp_b200.so")
WATCH = ["UTCHMMA", "UTCQMMA", "UTCBAR", "STTM", "LDTM", "UBLKCP", "UTMALDG", "LDGSTS", "SYNCS", "FFMA", "SHFL",
         "LDG", "STG", "LDS", "STS"]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            kernels[cur][m.group(1)] += 1
    names = {}
    for k in kernels:
        try:
            names[k] = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
        except OSError:
            names[k] = k
    print(f"# SASS opcode census of {os.path.basename(LIB)} (cuobjdump -sass, sm_100a)")
    print("# columns: " + " ".join(WATCH))
    total = collections.Counter()
    for k, c in kernels.items():
        total.update(c)
        if not any(c[w] for w in ("UTCHMMA", "UTCQMMA", "UBLKCP", "UTMALDG", "LDGSTS", "STTM", "LDTM")) \
                and "update" not in names[k] and "scatter" not in names[k]:
            continue
        nm = names[k].replace("stmp::", "").replace("(anonymous namespace)::", "")
        print(f"{nm[:120]}")
        print("    " + " ".join(f"{w}={c[w]}" for w in WATCH if c[w]))
    print("TOTAL " + " ".join(f"{w}={total[w]}" for w in WATCH))


if __name__ == "__main__":
    main()
