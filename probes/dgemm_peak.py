import torch, time, subprocess
torch.backends.cuda.matmul.allow_tf32 = False
for n in (4096, 8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10 if n < 16384 else 3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"cuBLAS DGEMM {n}^3: {2*n**3/best/1e9:.2f} TFLOP/s best ({best:.2f} ms)", flush=True)
# rank-k update shape like C2 step-1: (25600 x 128) @ (128 x 25600)
for (m, k) in ((25600, 128), (31500, 420)):
    a = torch.randn(m, k, dtype=torch.float64, device="cuda"); c = torch.randn(m, m, dtype=torch.float64, device="cuda")
    for _ in range(3): torch.addmm(c, a, a.t(), beta=1, alpha=-1, out=c)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): torch.addmm(c, a, a.t(), beta=1, alpha=-1, out=c)
    e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1) / 5
    print(f"cuBLAS rank-{k} update {m}x{m}: {2*m*m*k/ms/1e9:.2f} TFLOP/s ({ms:.2f} ms)", flush=True)
x = torch.empty(1 << 30, dtype=torch.uint8, device="cuda"); y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); [y.copy_(x) for _ in range(10)]; e1.record(); torch.cuda.synchronize()
print("copy GB/s", 2 * (1 << 30) * 10 / e0.elapsed_time(e1) / 1e6)
