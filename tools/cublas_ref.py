"""cuBLAS bf16 GEMM throughput on the same shapes (reference bar, diagnostic)."""
import sys, torch
for spec in sys.argv[1:]:
    M, N, K = (int(x) for x in spec.split(","))
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        c = a @ b.t()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        c = a @ b.t()
    e1.record(); torch.cuda.synchronize()
    print(spec, "cuBLAS TFLOP/s", round(2 * M * N * K * 10 / (e0.elapsed_time(e1) * 1e-3) / 1e12, 1))
