"""Opcode mix + stall samples of one kernel from an ncu report's SASS source page.
  ncu -i rep --page source --csv --print-source sass > x.csv ; python tools/ncu_opmix.py x.csv"""
import csv, collections, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iS = hdr.index('Source'); iE = hdr.index('Instructions Executed'); iW = hdr.index('Warp Stall Sampling (All Samples)')
op = collections.Counter(); samp = collections.Counter(); tot = 0; ts = 0
for r in rows[2:]:
    if len(r) <= iE:
        continue
    src = r[iS].strip(); n = int(r[iE] or 0); w = int(r[iW] or 0)
    m = re.match(r'(@!?U?P\w+\s+)?([A-Z0-9_.]+)', src)
    o = m.group(2).split('.')[0] if m else src
    op[o] += n; samp[o] += w; tot += n; ts += w
print('total warp instr', tot, 'samples', ts)
for o, n in op.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print('%-10s %6.2f%%  samples %5.1f%%' % (o, 100 * n / tot, 100 * samp[o] / ts))
