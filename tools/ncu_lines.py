"""Aggregate an ncu source page (cuda,sass csv) into the hottest CUDA lines."""
import csv, sys, collections
path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
cur_file = None
hdr = None
out = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    d = dict(zip(hdr[4:], r[4:]))
    try:
        samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    stalls = {k: v for k, v in d.items() if k.startswith("stall_")}
    out.append((samp, cur_file, r[0], r[1][:70], stalls, d.get("Instructions Executed", "")))
tot = sum(o[0] for o in out) or 1
out.sort(key=lambda o: -o[0])
print(f"total samples {tot}")
for samp, f, ln, src, stalls, ie in out[:top]:
    st = sorted(((int(v or 0), k[6:]) for k, v in stalls.items() if v not in ("", "0")), reverse=True)[:3]
    print(f"{100*samp/tot:5.1f}% {f}:{ln:5s} {src:70s} insts={ie} {st}")
