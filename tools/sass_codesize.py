"""Hot code size and samples per kernel phase from an ncu SASS source page (not part of the product).

    python tools/sass_codesize.py SASS.csv CUBIN KERNEL_MANGLED [depth]

Instructions executed >= 0.1 times per window count as hot code; each SASS
instruction is charged to its outermost inlined frame (the window-loop phase).
The cubin must be the measured build (cuobjdump -xelf all libotfgpu.so)."""
import csv, re, subprocess, collections, sys
path, cubin, kern = sys.argv[1:4]
rows = list(csv.reader(open(path)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if r and r[0].startswith("0x")]
txt = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout
line_of, cur, inside = {}, None, False
chain = []
for ln in txt.split("\n"):
    if ln.startswith("//--------------------- .text."):
        inside = ln.split(".text.")[1].split()[0] == kern; continue
    if not inside: continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        chain.append((m.group(1).split("/")[-1], int(m.group(2)))); continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(\S.*?);', ln)
    if m:
        if chain: cur = tuple(chain)
        chain = []
        if cur: line_of[int(m.group(1), 16)] = cur
W = 1024 * 29995.6
base = int(data[0]["Address"], 16)
depth = int(sys.argv[4]) if len(sys.argv) > 4 else 1
size = collections.Counter(); inst = collections.Counter()
for d in data:
    off = int(d["Address"], 16) - base
    e = int(d["Instructions Executed"] or 0) / W
    ch = line_of.get(off, (("?", 0),))
    key = ch[-depth:] if len(ch) >= depth else ch     # outermost `depth` frames
    key = key[0]
    if e >= 0.1:
        size[key] += 1
    inst[key] += e
src = {}
for k, n in size.most_common(30):
    f, l = k
    if f not in src:
        try: src[f] = open(__import__("os").environ.get("OTF_SRC", "paper_2603_08417_b200/csrc") + f"/{f}").read().split("\n")
        except Exception: src[f] = []
    t = src[f][l-1].strip()[:60] if 0 < l <= len(src[f]) else ""
    print(f"{n:5d} hot instrs ({n*16/1024:4.1f} KB)  {inst[k]:7.1f} exec/window  {f}:{l} {t}")
print("hot total", sum(size.values()))
