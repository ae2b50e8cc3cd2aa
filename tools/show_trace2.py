"""Per-chunk view of the projection trace (tools/trace_proj.py, STCA_TRACE)."""
import sys
import numpy as np
t = np.fromfile(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/trace_proj.bin', dtype=np.uint64).astype(np.int64)
ch = t[:4096].reshape(256, 16)
base = ch[0, 0]
print('gc   g1iss  g1done   g2iss  g2done | e_pre  e_gfull  e_ldtm  e_hfree  e_arrive')
for gc in range(0, 34):
    r = ch[gc]
    arr = [x for x in r[8:16] if x]
    f = lambda x: x - base if x else -1
    print(f'{gc:3d} {f(r[0]):7d} {f(r[1]):7d} {f(r[2]):7d} {f(r[3]):7d} | {f(r[7]):7d} {f(r[4]):7d} {f(r[5]):7d} {f(r[6]):7d} {max(arr) - base if arr else -1:7d}')
ln = t[4096:4096 + 64].reshape(8, 8)
print('LN [Y ready, Y released, stats done, staged | X: tma issued, landed, x_free, x_full]')
for l in ln[:5]:
    print('  ', [int(l[k] - base) if l[k] else -1 for k in (0, 3, 2, 1, 7, 4, 5, 6)])
