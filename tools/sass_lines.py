"""Map ncu per-SASS stall samples to CUDA source lines using nvdisasm -g output.
usage: sass_lines.py <ncu sass csv> <nvdisasm -g or -gi file (-gi: outermost call site)> <function mangled name> [topN]"""
import csv, re, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = [r for r in rows[2:] if len(r) == len(hdr)]
ix = {h: i for i, h in enumerate(hdr)}
S = ix['Warp Stall Sampling (All Samples)']
addrs = [int(r[ix['Address']], 16) for r in data]
base = min(addrs)
lines = open(sys.argv[2]).read().split('\n')
fn = sys.argv[3]
start = next(i for i, l in enumerate(lines) if l.startswith('.text.' + fn + ':'))
cur = None; off2line = {}
for l in lines[start + 1:]:
    if l.startswith('.text.'): break
    if l.lstrip().startswith('//## File'):
        locs = re.findall(r'"([^"]+)", line (\d+)', l)  # innermost first; with nvdisasm -gi the
        f, n = locs[-1]                                  # last one is the outermost call site
        cur = (f.split('/')[-1], int(n)); continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', l)
    if m and cur: off2line[int(m.group(1), 16)] = cur
agg = collections.defaultdict(float); stall = collections.defaultdict(lambda: collections.defaultdict(float))
sc = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
for r, a in zip(data, addrs):
    ln = off2line.get(a - base, ('?', 0))
    v = float(r[S] or 0); agg[ln] += v
    for h in sc: stall[ln][h] += float(r[ix[h]] or 0)
tot = sum(agg.values())
for ln, v in sorted(agg.items(), key=lambda x: -x[1])[:int(sys.argv[4]) if len(sys.argv) > 4 else 30]:
    top = sorted(stall[ln].items(), key=lambda x: -x[1])[:2]
    print(f"{v:7.0f} {100*v/tot:5.1f}% {ln[0]}:{ln[1]}  " + ", ".join(f"{k[6:]}={int(c)}" for k, c in top))
