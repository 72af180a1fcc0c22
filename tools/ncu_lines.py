"""Attribute ncu per-instruction counts (SASS source page CSV) to CUDA source lines
via nvdisasm --print-line-info of the same kernel (function-relative offsets).
  python tools/ncu_lines.py <sass.csv> <nvdisasm.dis> [top]"""
import csv, re, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iA = hdr.index('Address'); iE = hdr.index('Instructions Executed'); iW = hdr.index('Warp Stall Sampling (All Samples)')
iS = hdr.index('Source')
recs = [(int(r[iA], 16), int(r[iE] or 0), int(r[iW] or 0), r[iS]) for r in rows[2:] if len(r) > iE]
base = recs[0][0]
line_of = {}
cur = None
inl = None
for ln in open(sys.argv[2]):
    m = re.search(r'File "([^"]+)", line (\d+)', ln)
    if '//##' in ln and m:
        cur = int(m.group(2)) if m.group(1).endswith('kernels.cu') else -int(m.group(2))
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', ln)
    if m:
        line_of[int(m.group(1), 16)] = cur
agg = collections.Counter(); samp = collections.Counter()
tot = sum(r[1] for r in recs); ts = sum(r[2] for r in recs)
for a, n, w, s in recs:
    l = line_of.get(a - base)
    agg[l] += n; samp[l] += w
src = open('/root/repo/paper_2008_00216_b200/csrc/kernels.cu').read().split('\n')
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
print('total', tot, 'samples', ts)
for l, n in agg.most_common(top):
    print('%6.2f%% %6.2f%%  L%-5s %s' % (100 * n / tot, 100 * samp[l] / ts, l, (src[l - 1].strip()[:80] if l > 0 else ('<crt line %d>' % -l)) if l else ''))
if len(sys.argv) > 4 and sys.argv[4] == 'samples':
    print('--- by stall samples')
    for l, n in samp.most_common(top):
        print('%6.2f%% %6.2f%%  L%-5s %s' % (100 * agg[l] / tot, 100 * n / ts, l, (src[l - 1].strip()[:80] if l > 0 else ('<crt line %d>' % -l)) if l else ''))
