"""SASS mnemonic counts of the hot kernels (cuobjdump -sass of the built
library) — the static evidence that tcgen05 (UTCIMMA), TMA (UTMALDG/UTMASTG),
TMEM loads (LDTM) and DMMA are what the kernels run.

  python tools/sass_counts.py > profiles/r01_sass_counts.txt
"""
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1210_7683_b200", "libgwgrid_cuda.so")
KERNELS = ["_ZN3gwg16rotate_i8_kernelILi1EEEv14CUtensorMap_stS1_S1_S1_NS_6I8ArgsE",
           "_ZN3gwg19linear_solve_kernelILi4ELi2EEEv14CUtensorMap_stS1_S1_NS_7LinArgsE",
           "gls_sbr_kernel", "gls_grid_kernel", "rotate_kernel"]
KEEP = re.compile(r"^(UTC|UTMA|LDTM|DMMA|DFMA|I2F|LDG|STG|STS|SYNCS|UCGABAR|ELECT)")

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs, cur = {}, None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Za-z0-9_.]*)", line)
    if cur and m and KEEP.match(m.group(1)):
        funcs[cur][m.group(1)] += 1
print("# SASS mnemonic counts per hot kernel of paper_1210_7683_b200/libgwgrid_cuda.so "
      "(cuobjdump -sass, tools/sass_counts.py)")
print("# tcgen05 int8 MMA = UTCIMMA, TMA = UTMALDG/UTMASTG (+ multicast), TMEM loads = LDTM, "
      "FP64 tensor = DMMA.8x8x4")
for want in KERNELS:
    for name, cnt in funcs.items():
        if want == name or (want in name and name.startswith("_ZN3gwg") and
                            ("ILi4E" in name or "Sbr" in name or "rotate_kernel" in want)):
            print("## " + name)
            for op, c in cnt.most_common():
                print(f"{c:7d} {op}")
            break
