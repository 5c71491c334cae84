import torch, json
x = torch.empty(4 << 30 >> 3, dtype=torch.float64, device="cuda")
for _ in range(3): x.zero_()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): x.zero_()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(json.dumps({"memset_gbs": 4 * 2**30 / (ms * 1e-3) / 1e9, "ms": ms}))
y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
torch.cuda.synchronize()
e0.record()
for _ in range(10): y.copy_(x)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(json.dumps({"copy_gbs_rw": 2 * 4 * 2**30 / (ms * 1e-3) / 1e9, "ms": ms}))
