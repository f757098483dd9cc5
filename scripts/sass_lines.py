"""Per-source-line instruction counts of one kernel: joins `nvdisasm -g` line info with the
per-address 'Instructions Executed' of an ncu source-page CSV.
usage: sass_lines.py <nvdisasm -g output> <function mangled-name substring> <ncu source csv> <units>"""
import collections
import csv
import re
import sys

lines_txt, fname, src_csv, units = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
txt = open(lines_txt).read().split('\n')
start = next(i for i, l in enumerate(txt) if 'section' in l and '.text.' in l and fname in l)
addr2line, cur = {}, None
for l in txt[start + 1:]:
    if '.section' in l and '.text.' in l:
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.match(r'\s*/\*([0-9a-f]{4,5})\*/\s+(\S.*)', l)
    if m and cur:
        addr2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
seen, data = set(), []
for r in rows[2:]:
    if len(r) == len(hdr) and r[0].startswith('0x') and r[0] not in seen:
        seen.add(r[0])
        data.append(r)
ie, si = hdr.index('Instructions Executed'), hdr.index('Source')
base = int(data[0][0], 16)
agg, ops = collections.Counter(), collections.defaultdict(collections.Counter)
for r in data:
    ln = addr2line.get(int(r[0], 16) - base, ('?', 0))
    v = (int(r[ie]) if r[ie].isdigit() else 0) * 32 / units
    agg[ln] += v
    t = r[si].split()
    ops[ln][(t[1] if t[0].startswith('@') else t[0]).split('.')[0]] += v
srcs = {}
for f in {k[0] for k in agg}:
    for d in ('paper_1509_01149_b200/csrc/',):
        try:
            srcs[f] = open(d + f).read().split('\n')
        except OSError:
            pass
print('total per unit', round(sum(agg.values()), 1))
for (f, l), v in sorted(agg.items(), key=lambda x: -x[1])[:int(sys.argv[5]) if len(sys.argv) > 5 else 40]:
    s = srcs[f][l - 1].strip()[:58] if f in srcs else ''
    print(f'{v:6.1f} {f[:14]:14s}:{l:<4d} {s:58s} {dict((k, round(c, 1)) for k, c in ops[(f, l)].most_common(4))}')
