"""Per-kernel SASS instruction counts of libtmc.so that prove the tensor-core / TMEM / bulk-copy / MUFU
paths (cuobjdump -sass; no GPU needed).  Usage: python scripts/sass_counts.py [lib] > profiles/<round>_sass_counts.md"""
import collections, re, subprocess, sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1806_08593_b200/libtmc.so"
KEYS = ["UTCHMMA", "UTCBAR", "UTCCP", "LDTM", "STTM", "UBLKCP", "MUFU.EX2", "SYNCS", "FADD2", "F2FP", "HADD2.F32"]
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
counts, cur = collections.OrderedDict(), None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if cur and m:
        for k in KEYS:
            if m.group(1).startswith(k):
                counts[cur][k] += 1
print(f"SASS instruction counts per kernel of `{lib}` (static counts, `cuobjdump -sass`; kernels with any "
      "tcgen05 / TMEM / bulk-copy instruction)\n")
print("| kernel | " + " | ".join(KEYS) + " |")
print("|---" * (len(KEYS) + 1) + "|")
for f, c in counts.items():
    if any(c[k] for k in ("UTCHMMA", "LDTM", "UBLKCP", "UTCCP")):
        name = subprocess.run(["c++filt", f], capture_output=True, text=True).stdout.strip()
        print(f"| `{name.split('(')[0]}` | " + " | ".join(str(c[k]) for k in KEYS) + " |")
