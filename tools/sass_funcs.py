"""Static SASS instructions per enclosing source function (nvdisasm -g line info)."""
import re, sys, collections, subprocess
cub = sys.argv[1]
txt = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
cnt = collections.Counter(); cur = None
for line in txt.split("\n"):
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1), int(m.group(2))); continue
    if re.match(r'\s+/\*[0-9a-f]{4,}\*/\s+\S', line) and cur:
        cnt[cur] += 1
funcs = {}
for f in set(k[0] for k in cnt):
    try: src = open(f).read().split("\n")
    except Exception: continue
    starts = []
    for i, l in enumerate(src):
        m = re.match(r'^(?:static\s+)?(?:__host__\s+)?__device__[^(]*?(\w+)\s*\(', l) or \
            re.match(r'^OTF_HD\s+[^(]*?(\w+)\s*\(', l) or re.match(r'^__global__[^(]*?(\w+)\s*\(', l) or \
            re.match(r'^\s+__device__[^(]*?(\w+)\s*\(', l)
        if m: starts.append((i + 1, m.group(1)))
    funcs[f] = starts
agg = collections.Counter()
for (f, l), n in cnt.items():
    name = "?"
    for s, nm in funcs.get(f, []):
        if s <= l: name = nm
    agg[f.split("/")[-1] + ":" + name] += n
print("total", sum(cnt.values()))
for k, v in agg.most_common(45): print(v, k)
