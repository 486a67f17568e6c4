"""Aggregate an ncu `--page source --print-source cuda,sass --csv` dump per
source line: executed warp-instructions and stall samples.
usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > s.csv; python scripts/ncu_lines.py s.csv [top]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fpath = None; hdr = None
inst = collections.Counter(); samp = collections.Counter(); src = {}
stall = collections.defaultdict(collections.Counter)
for r in rows:
    if len(r) >= 2 and r[0] == "File Path": fpath = r[1].split("/")[-1]; continue
    if len(r) >= 2 and r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8: continue
    try: ln = int(r[0])
    except ValueError: continue
    key = (fpath, ln)
    src[key] = r[1].strip()[:70]
    try:
        inst[key] += int(r[7] or 0); samp[key] += int(r[4] or 0)
    except ValueError: pass
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try: stall[key][h[6:]] += int(r[i] or 0)
            except ValueError: pass
tot_i = sum(inst.values()); tot_s = sum(samp.values())
print(f"total warp-instr {tot_i:,}  samples {tot_s:,}")
for key, s in samp.most_common(top):
    st = ", ".join(f"{k}:{v}" for k, v in stall[key].most_common(3))
    print(f"{key[0][:18]:18s}:{key[1]:4d} samp {100*s/tot_s:5.1f}% inst {100*inst[key]/tot_i:5.1f}%  {src[key]:70s} [{st}]")
