"""cuBLAS (torch.matmul, bf16 in / fp32 accumulate) on the client-step GEMM shapes,
as a practical per-shape target for gemm_tc (tools/gemm_bench.py)."""
import torch

M, d, hid, V = 65536, 768, 3072, 50368
shapes = [("qkv/o fwd", M, d, d), ("w1 fwd", M, hid, d), ("w2 fwd", M, d, hid), ("head fwd", M, V, d),
          ("dX head", M, d, V), ("dW dxd", d, d, M), ("dW w1", d, hid, M), ("dW head", d, V, M)]
torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
for name, m, n, k in shapes:
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(k, n, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        c = a @ b
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"{name:10s} M={m:6d} N={n:6d} K={k:6d}  {ms*1e3:8.1f} us  {2*m*n*k/ms/1e9:7.1f} TF/s")
