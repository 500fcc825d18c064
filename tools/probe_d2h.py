import torch, time
n = 1 << 27  # 1 GiB of f64
d = torch.randn(n, dtype=torch.float64, device='cuda')
h = torch.empty(n, dtype=torch.float64).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for mode in ('one', 'two', 'four'):
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        if mode == 'one':
            h.copy_(d, non_blocking=True)
        else:
            k = 2 if mode == 'two' else 4
            c = n // k
            for i in range(k):
                st = s1 if i % 2 == 0 else s2
                with torch.cuda.stream(st):
                    h[i*c:(i+1)*c].copy_(d[i*c:(i+1)*c], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(mode, f"{8*n/dt/1e9:.1f} GB/s")
    h2 = h  # noqa
torch.cuda.synchronize(); t=time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); print('h2d', f"{8*n/(time.perf_counter()-t)/1e9:.1f} GB/s")
