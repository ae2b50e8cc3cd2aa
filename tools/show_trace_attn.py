"""Per-tile view of the attention trace (tools/trace_attn.py, STCA_TRACE_ATTN): work item 0."""
import sys
import numpy as np
t = np.fromfile(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/trace_attn.bin', dtype=np.uint64).astype(np.int64)
tr = t[:8192].reshape(512, 16)
nz = [j for j in range(480) if tr[j].any()]
base = min(x for j in nz for x in tr[j] if x)
print('j   tma   S:xful  S:pvok  S:cmt | PV:pful PV:cmt | sm:sful  max  bar  exp  Pst  arr0 arr4 arr7')
f = lambda x: x - base if x else -1
for j in nz[:40]:
    r = tr[j]
    print(f'{j:3d} {f(r[0]):6d} {f(r[1]):6d} {f(r[2]):6d} {f(r[3]):6d} | {f(r[4]):6d} {f(r[5]):6d} | '
          f'{f(r[6]):6d} {f(r[7]):6d} {f(r[8]):6d} {f(r[12]):6d} {f(r[13]):6d} {f(r[9]):6d} {f(r[10]):6d} {f(r[11]):6d}')
ep = t[7680:8192].reshape(64, 8)
print('item epilogues [load_u start, load_u done, pv waited, bar1, staged+o_free, bar2, copied]')
for k in range(64):
    if ep[k].any():
        print(k, [int(ep[k][e] - base) if ep[k][e] else -1 for e in (5, 6, 0, 1, 2, 3, 4)])
