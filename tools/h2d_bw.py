import torch
n = 660 * 1024 * 1024
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device='cuda')
for _ in range(3): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): d.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 10
print(f'H2D {n/1e9:.2f} GB in {t:.2f} ms = {n/t/1e6:.1f} GB/s')
s2 = torch.cuda.Stream()
half = n // 2
e0.record()
for _ in range(10):
    with torch.cuda.stream(s2):
        d[half:].copy_(h[half:], non_blocking=True)
    d[:half].copy_(h[:half], non_blocking=True)
torch.cuda.current_stream().wait_stream(s2)
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 10
print(f'H2D 2 streams: {n/t/1e6:.1f} GB/s')
