"""Static SASS instruction count per source line for one cubin (nvdisasm -g)."""
import re, sys, collections, subprocess
cub = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
cnt = collections.Counter(); cur = None
for line in txt.split("\n"):
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1), int(m.group(2))); continue
    if re.match(r'\s+/\*[0-9a-f]{4,}\*/\s+\S', line) and cur:
        cnt[cur] += 1
print("total", sum(cnt.values()))
by = collections.Counter()
for (f, l), n in cnt.items(): by[f.split("/")[-1]] += n
print(by.most_common())
for (f, l), n in cnt.most_common(top):
    try: src = open(f).read().split("\n")[l - 1].strip()[:90]
    except Exception: src = ""
    print(n, f.split("/")[-1], l, src)
