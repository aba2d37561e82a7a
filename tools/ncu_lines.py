"""Per-source-line warp-stall samples and executed instructions of one kernel in an ncu report,
mapped through `nvdisasm -g` of a locally built object (same source + flags => same SASS).

    python tools/ncu_lines.py report.ncu-rep paper_1111_6900_b200/csrc/_obj/product_run.o KERNEL_SUBSTR [--top N]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys


def main():
    rep, obj, kname = sys.argv[1:4]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
    src = list(csv.reader(io.StringIO(subprocess.run(
        ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
        text=True).stdout)))
    hdr = src[1]
    ix = {h: i for i, h in enumerate(hdr)}
    rows = []
    for r in src[2:]:  # first kernel of the report only (a later one repeats the header)
        if len(r) == len(hdr) and r[ix["Address"]] == "Address":
            break
        if len(r) == len(hdr):
            rows.append(r)
    base = int(rows[0][ix["Address"]], 16)
    samples = {int(r[ix["Address"]], 16) - base: int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in rows}
    execd = {int(r[ix["Address"]], 16) - base: int(r[ix["Instructions Executed"]] or 0) for r in rows}
    # SASS with line info from the local object
    cub = subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], capture_output=True, text=True,
                         cwd="/tmp")
    cubins = re.findall(r"(\S+\.cubin)", cub.stdout + cub.stderr)
    sass = ""
    for c in cubins:
        sass += subprocess.run(["nvdisasm", "-g", "-c", "/tmp/" + c], capture_output=True, text=True).stdout
    # pick the function
    funcs = re.split(r"\n\s*\.text\.", sass)
    body = next(f for f in funcs if kname in f.split(":")[0])
    line = None
    per_line = collections.Counter()
    per_line_ex = collections.Counter()
    for ln in body.splitlines():
        m = re.search(r'File "([^"]+)", line (\d+)', ln)
        if m and "//##" in ln:
            line = (m.group(1), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and line is not None:
            off = int(m.group(1), 16)
            per_line[line] += samples.get(off, 0)
            per_line_ex[line] += execd.get(off, 0)
    tot = sum(per_line.values()) or 1
    texts = {}
    print(f"{tot} samples mapped ({sum(samples.values())} in report)")
    for (fn, ln), s in per_line.most_common(top):
        if fn not in texts:
            try:
                texts[fn] = open(fn).read().splitlines()
            except OSError:
                texts[fn] = []
        t = texts[fn][ln - 1].strip()[:80] if ln - 1 < len(texts[fn]) else ""
        print(f"{100 * s / tot:5.1f}%  ex {per_line_ex[(fn, ln)]:>10d}  {os.path.basename(fn)}:{ln:<4d} {t}")


if __name__ == "__main__":
    main()
