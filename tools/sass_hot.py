"""Map an ncu SASS source page (per-instruction stall samples) to CUDA source lines.

    ncu -i REP --page source --csv --print-source sass > sass.csv
    python tools/sass_hot.py sass.csv CUBIN KERNEL_MANGLED [top]

The SASS rows are in address order; nvdisasm -gi of the same build gives each
instruction's source line (inlined frames: the innermost line).  Prints the
hottest lines with their top stall reasons, and the executed "hot code" size.
(Not part of the product.)
"""
import collections
import csv
import re
import subprocess
import sys

path, cubin, kern = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
SRC = sys.argv[5] if len(sys.argv) > 5 else "paper_2603_08417_b200/csrc"     # the measured build's sources
rows = list(csv.reader(open(path)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if r and r[0].startswith("0x")]
txt = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout
line_of, cur, opc = {}, None, {}
fresh = True
inside = False
for ln in txt.split("\n"):
    if ln.startswith("//--------------------- .text."):
        inside = ln.split(".text.")[1].split()[0] == kern
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        if fresh:                                      # the first location line of a block is the
            cur = (m.group(1).split("/")[-1], int(m.group(2)))   # innermost inlined frame
            fresh = False
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(\S.*?);', ln)
    if m:
        fresh = True
    if m and cur:
        off = int(m.group(1), 16)
        line_of[off] = cur
        opc[off] = m.group(2).split()[0].lstrip("@!P0123456789 ")
base = int(data[0]["Address"], 16)
stall_cols = [c for c in hdr if c.startswith("stall_")] or [c for c in hdr if c.lower().startswith("warp stall sampling (all")]
agg = collections.Counter()
why = collections.defaultdict(collections.Counter)
src = {}
hot = 0
mism = 0
for d in data:
    off = int(d["Address"], 16) - base
    samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    ex = int(d.get("Instructions Executed", "0") or 0)
    key = line_of.get(off, ("?", 0))
    if off in opc and not d["Source"].strip().startswith(opc[off][:3]) and opc[off][:3] not in d["Source"]:
        mism += 1
    agg[key] += samp
    if ex:
        hot += 1
for k in list(agg):
    pass
tot = sum(agg.values()) or 1
files = {}
print(f"total samples {tot}; {len(data)} SASS instructions, {hot} executed; opcode mismatches {mism}")
for (f, ln), s in agg.most_common(top):
    if f not in files:
        try:
            files[f] = open(subprocess.run(["bash", "-c", f"ls {SRC}/{f} 2>/dev/null || true"],
                                           capture_output=True, text=True).stdout.strip()).read().split("\n")
        except Exception:
            files[f] = []
    text = files[f][ln - 1].strip()[:80] if 0 < ln <= len(files[f]) else ""
    print(f"{100 * s / tot:5.1f}% {f}:{ln:<5d} {text}")
