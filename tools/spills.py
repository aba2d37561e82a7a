"""Dev: registers and spills per kernel instantiation of a CUDA source (ptxas -v).
python tools/spills.py paper_1111_6900_b200/csrc/product_tc2.cu [--all]"""
import re
import subprocess
import sys

src = sys.argv[1]
out = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                      "--expt-relaxed-constexpr", "-Xptxas", "-v", "-c", src, "-o", "/tmp/_spills.o"],
                     capture_output=True, text=True).stderr
name, spill = None, (0, 0)
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"gf2e::\(anonymous namespace\)::", "", name).split("(")[0]
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        spill = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        if spill != (0, 0) or "--all" in sys.argv:
            print(f"{name:60s} regs {m.group(1):>4s} spill st/ld {spill}")
        name, spill = None, (0, 0)
