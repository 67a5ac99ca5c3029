import ctypes as C, sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2411_02908_b200 import _capi as A
lib = A.lib()
def run(M, N, K, ak, bk, epi, cbf):
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    b = (torch.randn(K, N, device="cuda", generator=g) * 0.05).bfloat16()
    A_st = a if ak else a.t().contiguous()
    B_st = b.t().contiguous() if bk else b
    bias = torch.randn(N, device="cuda")
    resid = torch.randn(M, N, device="cuda") if epi == 3 else None
    out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16 if cbf else torch.float32)
    ms, err = C.c_double(), A.photon_err()
    rc = lib.photon_debug_gemm(1, M, N, K, A_st.data_ptr(), K if ak else M, int(ak), B_st.data_ptr(), K if bk else N, int(bk), 1,
                               out.data_ptr(), N, int(cbf), epi, bias.data_ptr(), resid.data_ptr() if resid is not None else None, None, 1, C.byref(ms), C.byref(err))
    torch.cuda.synchronize()
    ref = a[:64].float() @ b.float()
    got = out[:64].float()
    print(M, N, K, ak, bk, epi, cbf, "rc", rc, err.msg, "ms %.3f" % ms.value, "max|out| %.3g" % out.float().abs().max().item(), "err0 %.3g" % (got - (ref if epi == 0 else got)).abs().max().item(), flush=True)
for args in [(65536, 768, 3072, 1, 0, 3, 0), (4096, 768, 3072, 1, 0, 3, 0), (65536, 768, 3072, 1, 0, 0, 0), (16384, 768, 50368, 1, 1, 0, 0), (4096, 768, 50368, 1, 1, 0, 0), (16384, 768, 8192, 1, 1, 0, 0), (768, 50368, 16384, 0, 0, 0, 0), (768, 50368, 4096, 0, 0, 0, 0), (768, 8192, 16384, 0, 0, 0, 0)]:
    run(*args)
