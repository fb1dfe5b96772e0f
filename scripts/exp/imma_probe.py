import torch, time
torch.backends.cuda.matmul.allow_tf32 = False
def bench(f, reps=5):
    f(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): f()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
n, M = 1100000, 912
for K in (912, 912*4, 912*7):
    a = torch.randint(-127, 127, (n, K), dtype=torch.int8, device='cuda')
    b = torch.randint(-127, 127, (K, M), dtype=torch.int8, device='cuda').t().contiguous().t()
    ms = bench(lambda: torch._int_mm(a, b))
    print(f"int8 [{n}x{K}]@[{K}x{M}] {ms:.2f} ms  {2*n*K*M/ms/1e9:.0f} TOPS", flush=True)
    del a, b
# small-output long-k shape: [912 x k] @ [k x 912]
for k in (131072, 1100000//8*8):
    a = torch.randint(-127, 127, (M, k), dtype=torch.int8, device='cuda')
    b = torch.randint(-127, 127, (k, M), dtype=torch.int8, device='cuda').t().contiguous().t()
    ms = bench(lambda: torch._int_mm(a, b))
    print(f"int8 [{M}x{k}]@[{k}x{M}] {ms:.3f} ms  {2*k*M*M/ms/1e9:.0f} TOPS", flush=True)
a = torch.randn(n, M, dtype=torch.float64, device='cuda'); b = torch.randn(M, M, dtype=torch.float64, device='cuda')
ms = bench(lambda: a @ b)
print(f"fp64 [{n}x{M}]@[{M}x{M}] {ms:.2f} ms {2*n*M*M/ms/1e9:.0f} GFLOPs")
x = torch.randn(n, 8*M//8, dtype=torch.float64, device='cuda')
ms = bench(lambda: x.to(torch.int8))
print(f"convert f64->i8 {n}x{M}: {ms:.2f} ms")
