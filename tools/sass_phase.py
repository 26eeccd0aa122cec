"""Stall samples and executed instructions per source line (outer: the window-loop phase; inner: the innermost inlined line) from an ncu SASS source page (not part of the product).

    python tools/sass_phase.py SASS.csv CUBIN KERNEL_MANGLED outer|inner [top]"""
import csv, re, subprocess, collections, sys
path, cubin, kern = sys.argv[1:4]
outer = sys.argv[4] == "outer" if len(sys.argv) > 4 else True
rows = list(csv.reader(open(path)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if r and r[0].startswith("0x")]
txt = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout
line_of, cur, inside, fresh = {}, None, False, True
for ln in txt.split("\n"):
    if ln.startswith("//--------------------- .text."):
        inside = ln.split(".text.")[1].split()[0] == kern; continue
    if not inside: continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        loc = (m.group(1).split("/")[-1], int(m.group(2)))
        if outer: cur = loc
        elif fresh: cur = loc; fresh = False
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(\S.*?);', ln)
    if m:
        fresh = True
        if cur: line_of[int(m.group(1), 16)] = cur
base = int(data[0]["Address"], 16)
samp = collections.Counter(); inst = collections.Counter(); thr = collections.Counter()
for d in data:
    off = int(d["Address"], 16) - base
    k = line_of.get(off, ("?", 0))
    samp[k] += int(d["Warp Stall Sampling (All Samples)"] or 0)
    inst[k] += int(d["Instructions Executed"] or 0)
    thr[k] += int(d["Thread Instructions Executed"] or 0)
ts, ti = sum(samp.values()), sum(inst.values())
src = {}
for k, s in samp.most_common(int(sys.argv[5]) if len(sys.argv) > 5 else 25):
    f, l = k
    if f not in src:
        try: src[f] = open(__import__("os").environ.get("OTF_SRC", "paper_2603_08417_b200/csrc") + f"/{f}").read().split("\n")
        except Exception: src[f] = []
    t = src[f][l-1].strip()[:60] if 0 < l <= len(src[f]) else ""
    print(f"{100*s/ts:5.1f}% samp {100*inst[k]/ti:5.1f}% inst  {thr[k]/max(1,inst[k]):5.1f} thr  {f}:{l} {t}")
print("total inst", ti)
