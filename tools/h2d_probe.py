import time, numpy as np, torch
x = np.random.rand(1000000, 50)
torch.cuda.synchronize()
for _ in range(2):
    t = torch.as_tensor(x, device='cuda'); torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter(); t = torch.as_tensor(x, device='cuda'); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
print('pageable as_tensor 400 MB: ms', [round(v * 1e3, 1) for v in ts], 'GB/s', round(0.4 / sorted(ts)[2], 1))
p = torch.empty((1000000, 50), dtype=torch.float64, pin_memory=True)
ts = []
for _ in range(5):
    t0 = time.perf_counter(); p.copy_(torch.from_numpy(x)); t = p.to('cuda', non_blocking=True); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
print('host copy into pinned + H2D: ms', [round(v * 1e3, 1) for v in ts])
ts = []
for _ in range(5):
    t0 = time.perf_counter(); t = p.to('cuda', non_blocking=True); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
print('pinned H2D only: ms', [round(v * 1e3, 1) for v in ts], 'GB/s', round(0.4 / sorted(ts)[2], 1))
