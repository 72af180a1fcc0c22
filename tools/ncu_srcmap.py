"""Attribute an ncu SASS source-page CSV (ncu -i rep --page source --csv --print-source sass) to
CUDA source lines through nvdisasm --print-line-info -fun <symbol index> of the same cubin.
  python tools/ncu_srcmap.py <sass.csv> <nvdisasm.dis> [top]"""
import collections
import csv
import os
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iA, iE = hdr.index('Address'), hdr.index('Instructions Executed')
iW = hdr.index('Warp Stall Sampling (All Samples)')
recs = [(int(r[iA], 16), int(r[iE] or 0), int(r[iW] or 0)) for r in rows[2:] if len(r) > iE]
base = recs[0][0]
line_of, cur = {}, None
for ln in open(sys.argv[2]):
    m = re.search(r'File "([^"]+)", line (\d+)', ln)
    if '//##' in ln and m:
        cur = (m.group(1), int(m.group(2)))
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', ln)
    if m:
        line_of[int(m.group(1), 16)] = cur
agg, samp = collections.Counter(), collections.Counter()
tot, ts = sum(r[1] for r in recs), sum(r[2] for r in recs)
for a, n, w in recs:
    key = line_of.get(a - base)
    agg[key] += n
    samp[key] += w
cache = {}


def text(key):
    if not key:
        return '?'
    f, l = key
    if f not in cache:
        p = f if os.path.exists(f) else os.path.join('paper_2008_00216_b200/csrc', os.path.basename(f))
        cache[f] = open(p).read().split('\n') if os.path.exists(p) else []
    src = cache[f]
    return '%s:%d %s' % (os.path.basename(f), l, src[l - 1].strip()[:80] if l - 1 < len(src) else '')


top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
print('total warp-instructions', tot, 'stall samples', ts)
print('-- by executed instructions')
for k, n in agg.most_common(top):
    print('%6.2f%% %6.2f%%  %s' % (100 * n / tot, 100 * samp[k] / ts, text(k)))
print('-- by stall samples')
for k, n in samp.most_common(top):
    print('%6.2f%% %6.2f%%  %s' % (100 * agg[k] / tot, 100 * n / ts, text(k)))
