"""Summarise an ncu source-page SASS csv: stall mix, opcode mix, hot blocks."""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
S = lambda r, k: int(r[idx[k]] or 0)
tot = sum(S(r, 'Warp Stall Sampling (All Samples)') for r in data)
ti = sum(S(r, 'Instructions Executed') for r in data)
print('samples', tot, 'warp insts', ti)
reasons = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
agg = {h: sum(S(r, h) for r in data) for h in reasons}
print([(k, f'{v/tot:.1%}') for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]])
c = Counter()
for r in data:
    op = r[idx['Source']].split()
    if not op:
        continue
    o = op[0] if not op[0].startswith('@') else op[1]
    c[o.split('.')[0]] += S(r, 'Instructions Executed')
print([(k, f'{v/ti:.1%}') for k, v in c.most_common(14)])
blocks, cur = [], None
for r in data:
    e = S(r, 'Instructions Executed'); s = S(r, 'Warp Stall Sampling (All Samples)')
    if cur and cur[0] == e:
        cur[1] += 1; cur[2] += s; cur[4].append(r[idx['Source']][:38])
    else:
        cur = [e, 1, s, r[idx['Address']][-5:], [r[idx['Source']][:38]]]; blocks.append(cur)
blocks.sort(key=lambda b: -b[0] * b[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
for b in blocks[:n]:
    print(b[3], 'exec', b[0], 'ninst', b[1], 'total', b[0] * b[1], f'({b[0]*b[1]/ti:.1%})', 'stall', b[2], b[4][:3])
