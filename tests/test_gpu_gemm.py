"""tcgen05 GEMM (and the SIMT GEMM) vs a plain PyTorch fp32 reference of the same
op.  Inputs are bf16-representable, so the only differences are fp32
accumulation order (fp32 out: rel <= 1e-4 of the output scale) and the final
bf16 rounding (bf16 out: rel <= 1e-2)."""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _run(impl, M, N, K, a_kmajor, b_kmajor, epi, c_bf16, seed=0):
    from paper_2411_02908_b200 import _capi as A

    g = torch.Generator(device="cuda").manual_seed(seed)
    dev = "cuda"
    # logical A [M,K], B [K,N]; stored per layout
    a = torch.randn(M, K, device=dev, generator=g).bfloat16()
    b = torch.randn(K, N, device=dev, generator=g).bfloat16() * 0.1
    A_st = a.contiguous() if a_kmajor else a.t().contiguous()       # [M,K] or [K,M]
    B_st = b.t().contiguous() if b_kmajor else b.contiguous()       # [N,K] or [K,N]
    lda = K if a_kmajor else M
    ldb = K if b_kmajor else N
    bias = torch.randn(N, device=dev, generator=g) * 0.5
    resid = torch.randn(M, N, device=dev, generator=g)
    cdt = torch.bfloat16 if c_bf16 else torch.float32
    Cbuf = torch.randn(M, N, device=dev, generator=g).to(cdt)
    aux = (torch.randn(M, N, device=dev, generator=g)).bfloat16()
    C0 = Cbuf.clone()
    aux0 = aux.clone()
    ms = C.c_double()
    err = A.photon_err()
    rc = A.lib().photon_debug_gemm(impl, M, N, K, A_st.data_ptr(), lda, int(a_kmajor),
                                   B_st.data_ptr(), ldb, int(b_kmajor), 1, Cbuf.data_ptr(), N,
                                   int(c_bf16), epi, bias.data_ptr(), resid.data_ptr(),
                                   aux.data_ptr(), 1, C.byref(ms), C.byref(err))
    assert rc == 0, err.msg
    torch.cuda.synchronize()
    acc = a.float() @ b.float()
    if epi == 0:
        ref = acc
    elif epi == 1:
        ref = C0.float() + acc
    elif epi == 2:
        ref = acc + bias
    elif epi == 3:
        ref = resid + (acc + bias)
    elif epi == 4:  # C = gelu(u), aux = gelu'(u) for the backward, u = acc + bias
        pre = acc + bias
        ref = torch.nn.functional.gelu(pre)
        cdf = 0.5 * (1 + torch.erf(pre * 0.7071067811865476))
        pdf = 0.3989422804014327 * torch.exp(-0.5 * pre * pre)
        assert torch.allclose(aux.float(), cdf + pre * pdf, rtol=1e-2, atol=1e-2)
    elif epi == 5:  # C = acc * aux
        ref = acc * aux0.float()
    out = Cbuf.float()
    scale = ref.abs().max().item() + 1e-6
    tol = 1e-2 if c_bf16 else 1e-4
    err_max = (out - ref).abs().max().item() / scale
    assert err_max <= tol, (impl, M, N, K, a_kmajor, b_kmajor, epi, c_bf16, err_max)
    return ms.value


SHAPES = [(128, 256, 64), (256, 768, 768), (200, 72, 40), (64, 56, 8), (296, 520, 200),
          (768, 768, 8192)]


@pytest.mark.parametrize("impl", [1, 0])
@pytest.mark.parametrize("a_kmajor", [True, False])
@pytest.mark.parametrize("b_kmajor", [True, False])
@pytest.mark.parametrize("shape", SHAPES)
def test_gemm_layouts_store_f32(impl, a_kmajor, b_kmajor, shape):
    M, N, K = shape
    if impl == 0 and K > 1000:
        pytest.skip("SIMT path: long-K case covered by the tcgen05 path")
    _run(impl, M, N, K, a_kmajor, b_kmajor, epi=0, c_bf16=False)


@pytest.mark.parametrize("epi,c_bf16", [(0, True), (1, False), (2, True), (2, False), (3, False),
                                        (4, True), (5, True)])
@pytest.mark.parametrize("shape", [(256, 768, 768), (136, 200, 72)])
def test_gemm_epilogues(epi, c_bf16, shape):
    M, N, K = shape
    _run(1, M, N, K, True, False, epi, c_bf16)
    _run(0, M, N, K, True, False, epi, c_bf16)


@pytest.mark.parametrize("M,N,bf", [(4096, 50368, 1), (1000, 8192, 1), (300, 768, 1), (257, 3072, 0),
                                    (2048, 16384, 1), (65536, 768, 1), (8192, 3072, 1),
                                    (5000, 256, 1), (3001, 1032, 1)])
def test_bias_grad_colsum(M, N, bf):
    # the head bias (N = V) takes the whole-row shared-memory kernel, moderate
    # widths the row-slot kernel, small inputs the strip kernel; all against a
    # float64 torch column sum
    import ctypes as C

    from paper_2411_02908_b200 import _capi as A

    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(M, N, device="cuda", generator=g)
    x = x.bfloat16() if bf else x
    out = torch.empty(N, device="cuda")
    ms = C.c_double()
    err = A.photon_err()
    assert A.lib().photon_debug_colsum(x.data_ptr(), bf, M, N, out.data_ptr(), C.byref(ms),
                                       C.byref(err)) == 0, err.msg
    torch.cuda.synchronize()
    ref = x.double().sum(0)
    assert (out.double() - ref).abs().max().item() <= 1e-3 * (1 + ref.abs().max().item())


def test_k_concatenated_gemm(monkeypatch):
    # photon_debug_gemm with PHOTON_DEBUG_NSEG=3 repeats (A, B) as three K
    # segments into one accumulator: C = 3 A B (the LayerNorm-1 dX contraction
    # dv Wv^T + dk Wk^T + dq Wq^T uses the same kernel path with distinct pairs)
    import ctypes as C

    from paper_2411_02908_b200 import _capi as A

    M, N, K = 512, 768, 256
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    b = torch.randn(N, K, device="cuda", generator=g).bfloat16()  # K-major B (dX layout)
    c = torch.zeros(M, N, device="cuda")
    ms = C.c_double()
    err = A.photon_err()
    monkeypatch.setenv("PHOTON_DEBUG_NSEG", "3")
    rc = A.lib().photon_debug_gemm(1, M, N, K, a.data_ptr(), K, 1, b.data_ptr(), K, 1, 1,
                                   c.data_ptr(), N, 0, 0, None, None, None, 1, C.byref(ms),
                                   C.byref(err))
    assert rc == 0, err.msg
    torch.cuda.synchronize()
    ref = 3.0 * (a.float() @ b.float().t())
    assert (c - ref).abs().max().item() <= 1e-3 * ref.abs().max().item()
