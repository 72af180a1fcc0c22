"""Aggregate ncu SASS source-page counts by CUDA device function (kernels.cu) or crt header line.
  python tools/ncu_funcs.py <sass.csv> <nvdisasm.dis> [top]"""
import csv, re, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iA = hdr.index('Address'); iE = hdr.index('Instructions Executed')
iW = hdr.index('Warp Stall Sampling (All Samples)'); iS = hdr.index('Source')
recs = [(int(r[iA], 16), int(r[iE] or 0), int(r[iW] or 0), r[iS]) for r in rows[2:] if len(r) > iE]
base = recs[0][0]
line_of = {}
cur = None
for ln in open(sys.argv[2]):
    m = re.search(r'File "([^"]+)", line (\d+)', ln)
    if '//##' in ln and m:
        cur = int(m.group(2)) if m.group(1).endswith('kernels.cu') else -int(m.group(2))
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', ln)
    if m:
        line_of[int(m.group(1), 16)] = cur
src = open('/root/repo/paper_2008_00216_b200/csrc/kernels.cu').read().split('\n')
funcs = []
for i, l in enumerate(src, 1):
    m = re.search(r'(?:__device__|__global__).*?\b(\w+)\s*\(', l)
    if m and not l.strip().startswith('//'):
        funcs.append((i, m.group(1)))


def fn(l):
    if l is None:
        return 'None'
    if l < 0:
        return 'crt%d' % -l
    best = '?'
    for i, n in funcs:
        if i <= l:
            best = n
    return best


agg = collections.Counter(); smp = collections.Counter(); ops = collections.defaultdict(collections.Counter)
tot = sum(r[1] for r in recs); ts = sum(r[2] for r in recs)
for a, n, w, s in recs:
    f = fn(line_of.get(a - base)); agg[f] += n; smp[f] += w
    toks = s.split()
    op = (toks[1] if toks and toks[0].startswith('@') and len(toks) > 1 else (toks[0] if toks else ''))
    ops[f][op.split('.')[0]] += n
print('total warp instr', tot, 'samples', ts)
for f, n in agg.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 25):
    if n == 0:
        continue
    print('%6.2f%% %6.2f%% %-22s %s' % (100 * n / tot, 100 * smp[f] / max(ts, 1), f,
                                        ', '.join('%s:%.1f' % (o, 100 * c / n) for o, c in ops[f].most_common(6))))
