"""Print the clock64 trace written by STCA_TRACE (tools/trace_proj.py)."""
import sys
import numpy as np
t = np.fromfile(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/trace_proj.bin', dtype=np.uint64).astype(np.int64)
ch = t[:4096].reshape(256, 16)[:64]
ln = t[4096:4096 + 32].reshape(4, 8)
base = ch[0, 0]
names = ['mma_wfull', 'mma_g1done', 'mma_hful2', 'mma_g2done', 'e0_gfull', 'e0_ldtm', 'e0_hfree', 'tma_iss'] + [f'arr_w{w}' for w in range(8)]
print('gc  ' + ' '.join(f'{n:>9s}' for n in names))
for gc in list(range(0, 12)) + list(range(28, 32)):
    print(f'{gc:3d} ' + ' '.join(f'{(ch[gc, k] - base) if ch[gc, k] else -1:9d}' for k in range(16)))
print('LN [Y ready, stats done, staged]')
for l in ln:
    print('  ', [int(l[k] - base) for k in (0, 2, 1)])
