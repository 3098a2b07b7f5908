"""Attribute an ncu source-page SASS listing to CUDA source lines.

    ncu -i REP --page source --csv --print-source sass > src.csv
    cuobjdump -xelf all paper_2603_09038_b200/_build/pa_p4.o   # -> pa_inst.sm_100a.cubin
    nvdisasm -g pa_inst.sm_100a.cubin > sass.txt
    python tools/sass_attr.py MANGLED_KERNEL sass.txt src.csv NUM_ELEMENTS [TOP]

Joins ncu's per-address "Instructions Executed" / "L1 Wavefronts Shared" with
nvdisasm's line table (the library is built with -lineinfo) and prints warp
instructions and shared wavefronts per element for the hottest source lines,
with their opcode mix (how the precomputed-gather change, DESIGN.md §4.3,
was found).
"""
import collections
import csv
import re
import sys

F, sassf, csvf, nel = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
lines=open(sassf).read().split('\n')
start=[i for i,l in enumerate(lines) if l.startswith('//--------------------- .text.'+F)][0]
cur=None; src={}
for l in lines[start+1:]:
    if l.startswith('//---------------------'): break
    m=re.search(r'//## File "([^"]+)", line (\d+)',l)
    if m: cur=(m.group(1).split('/')[-1],int(m.group(2))); continue
    m=re.search(r'/\*([0-9a-f]{4,})\*/\s+(.*?);',l)
    if m: src[int(m.group(1),16)]=(cur,m.group(2))
rows=list(csv.reader(open(csvf)))
h=rows[1]; iA=h.index('Address'); iE=h.index('Instructions Executed'); iW=h.index('L1 Wavefronts Shared')
base=int(rows[2][iA],16)
agg=collections.Counter(); ops=collections.defaultdict(collections.Counter); wf=collections.Counter()
for r in rows[2:]:
    a=int(r[iA],16)-base; n=int(r[iE] or 0)
    if a in src:
        loc,ins=src[a]
        agg[loc]+=n; wf[loc]+=int(r[iW] or 0)
        t=ins.split(); o=t[1] if t[0].startswith('@') else t[0]
        ops[loc][o.split('.')[0]]+=n
tot=sum(agg.values())
print('total/el', tot/nel)
for loc,n in agg.most_common(int(sys.argv[5]) if len(sys.argv)>5 else 40):
    print(f"{n/nel:7.1f} wf {wf[loc]/nel:6.1f} {loc}  {dict(ops[loc].most_common(5))}")
