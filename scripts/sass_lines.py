"""Static SASS size per source line for one kernel:
nvdisasm -g -c X.cubin > all.sass; python scripts/sass_lines.py all.sass <kernel-substring> [top]"""
import collections, re, sys
lines = open(sys.argv[1]).read().split("\n")
want = sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cur = None; fn = None; src = {}
cnt = collections.Counter()
for line in lines:
    m = re.match(r"\.text\.(\S+):", line)
    if m:
        fn = m.group(1); continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2))); continue
    if fn and want in fn and re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
        cnt[cur] += 1
tot = sum(cnt.values())
print(f"{want}: {tot} instructions = {tot * 16 / 1024:.1f} KB")
files = {}
for (f, l), c in cnt.most_common(top):
    if f not in files:
        import os
        for d in ("paper_2106_14995_b200/csrc", "/usr/local/cuda/include", "/usr/local/cuda/include/crt"):
            p = os.path.join(d, f)
            if os.path.exists(p):
                files[f] = open(p).read().split("\n"); break
    s = files.get(f, [""] * (l + 1))[l - 1].strip()[:80] if f in files else ""
    print(f"{c:5d} {100 * c / tot:5.1f}%  {f}:{l}  {s}")
