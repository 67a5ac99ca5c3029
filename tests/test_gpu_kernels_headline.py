"""The kernel instances the 125M headline config runs, at its shapes, each
against a plain PyTorch fp32/f64 reference of the same op (through the C ABI's
debug hooks, which call exactly what the engine calls):

  * softmax cross-entropy at V = 50,368 (tensor.cpp:544-603): the persistent
    pipelined kernel (two 100 KB shared-memory row buffers, refills when
    M > 148), forward-only, target padding, NaN rows, with the head-bias
    column sums accumulated in tensor memory inside the same pass (fp32, before
    the bf16 rounding) and, where that does not apply, the column-sum kernels;
  * LayerNorm forward / backward at d = 768 (the register-resident NV = 6
    kernels) and d = 4,096 (the row-split WPR = 8 kernels of the 7B config)
    (tensor.cpp:322-394);
  * tcgen05 GEMMs at M = 65,536 and the head's N = 50,368, where the grouped
    raster has many bands (num_m > group_m), checked on sampled rows spread
    over every band (tensor.cpp:152-207).

Tolerances (stated per check below): fp32 outputs rel 1e-4 of the output
scale; bf16 outputs one bf16 rounding (rel 1e-2 of the scale); row losses rel
1e-5; the head-bias column sums (fp32, over the unrounded gradient values,
fused into the cross-entropy pass) rel 3e-4 of the largest column sum; LayerNorm
column sums rel 1e-4.
"""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

V125 = 50368


def _A():
    from paper_2411_02908_b200 import _capi as A

    return A


# ---------------------------------------------------------------------------
# cross-entropy (+ fused head-bias gradient)
# ---------------------------------------------------------------------------
def _ce_case(M, V, write_grad, with_bias, seed=0, pad_rows=(), nan_row=None, fused_bias=True):
    A = _A()
    g = torch.Generator(device="cuda").manual_seed(seed)
    logits = (torch.randn(M, V, device="cuda", generator=g) * 2.0).bfloat16()
    tgt = torch.randint(0, V, (M,), device="cuda", generator=g, dtype=torch.int32)
    for r in pad_rows:
        tgt[r] = -1
    if nan_row is not None:
        logits[nan_row, 7] = float("nan")
    count = int((tgt >= 0).sum().item())
    inv = 1.0 / max(count, 1)
    x = logits.float()
    rowloss = torch.zeros(M, device="cuda", dtype=torch.float64)
    dbias = torch.zeros(V, device="cuda") if with_bias else None
    buf = logits.clone()
    ms = C.c_double()
    err = A.photon_err()
    rc = A.lib().photon_debug_ce(buf.data_ptr(), 1, tgt.data_ptr(), M, V, C.c_float(inv),
                                 rowloss.data_ptr(), int(write_grad),
                                 dbias.data_ptr() if with_bias else None, C.byref(ms),
                                 C.byref(err))
    assert rc == 0, err.msg
    torch.cuda.synchronize()
    # reference (f64): loss_r = logsumexp - l[t]; dl = (softmax - onehot) / count
    xd = x.double()
    lse = torch.logsumexp(xd, dim=1)
    valid = tgt >= 0
    tl = tgt.clamp(min=0).long()
    ref_loss = torch.where(valid, lse - xd.gather(1, tl[:, None])[:, 0], torch.zeros_like(lse))
    ok = torch.ones(M, dtype=torch.bool, device="cuda")
    if nan_row is not None:
        assert torch.isnan(rowloss[nan_row]).item()
        ok[nan_row] = False
    err_l = ((rowloss - ref_loss).abs() / ref_loss.abs().clamp(min=1.0))[ok].max().item()
    assert err_l <= 1e-5, err_l
    if not write_grad:
        assert torch.equal(buf, logits)  # eval: logits untouched
        return ms.value
    p = torch.softmax(xd, dim=1)
    onehot = torch.zeros_like(p)
    onehot[valid, tl[valid]] = 1.0
    ref_g = (p - onehot) * inv
    ref_g[~valid] = 0.0
    got = buf.double()
    scale = ref_g[ok].abs().max().item()
    # one bf16 rounding of each gradient value (rel 2^-8), abs floor for p ~ 0
    d = (got - ref_g)[ok].abs()
    assert (d <= 8e-3 * ref_g[ok].abs() + 1e-6 * scale).all(), d.max().item()
    if with_bias and nan_row is None:  # (a NaN row makes every column sum NaN, as in f64)
        # fused: fp32 sums of the unrounded values (rel 3e-4); the separate
        # column-sum pass adds the bf16-rounded values (rel 2^-9 each)
        ref_b = ref_g[ok].sum(0)
        eb = (dbias.double() - ref_b).abs().max().item() / (ref_b.abs().max().item() + 1e-30)
        assert eb <= (3e-4 if fused_bias else 2e-3), eb
    return ms.value


def test_ce_head_shape_with_bias():
    # M = 1,024 > 148: every persistent CTA refills its row buffers
    _ce_case(1024, V125, True, True)


def test_ce_head_shape_padding_and_nan():
    # target < 0 rows contribute no loss and no gradient (tensor.cpp:569-600);
    # a NaN logit makes that row's loss NaN (DivergenceError upstream)
    _ce_case(1024, V125, True, True, seed=3, pad_rows=(0, 5, 777, 1023), nan_row=300)


@pytest.mark.parametrize("M", [1024, 150])
def test_ce_head_shape_pipe_kernel(M):
    # M < 2 x 148 included (some CTAs get one row, none a refill)
    _ce_case(M, V125, True, False, seed=1)


def test_ce_head_shape_small_m_with_bias():
    # M = 200: some persistent CTAs own two rows, most one
    _ce_case(200, V125, True, True, seed=2)


def test_ce_forward_only():
    _ce_case(512, V125, False, False, seed=4)


def test_ce_odd_vocab_with_bias():
    # V / 8 odd
    _ce_case(640, 8 * 1001, True, True, seed=5)


# ---------------------------------------------------------------------------
# LayerNorm forward / backward
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("d", [768, 4096])
@pytest.mark.parametrize("y_bf16", [1, 0])
def test_layernorm_headline_widths(d, y_bf16):
    A = _A()
    M = 4096
    g = torch.Generator(device="cuda").manual_seed(d + y_bf16)
    x = torch.randn(M, d, device="cuda", generator=g) * 1.5 + 0.3
    gain = 1.0 + 0.1 * torch.randn(d, device="cuda", generator=g)
    bias = 0.1 * torch.randn(d, device="cuda", generator=g)
    tdt = torch.bfloat16 if y_bf16 else torch.float32
    dy = torch.randn(M, d, device="cuda", generator=g).to(tdt)  # the dX GEMMs' output type
    dres = torch.randn(M, d, device="cuda", generator=g)
    y = torch.empty(M, d, device="cuda", dtype=tdt)
    mean = torch.empty(M, device="cuda")
    rstd = torch.empty(M, device="cuda")
    dx = torch.empty(M, d, device="cuda")
    dxT = torch.empty(M, d, device="cuda", dtype=tdt)
    dgain = torch.empty(d, device="cuda")
    dbias = torch.empty(d, device="cuda")
    dsum = torch.empty(d, device="cuda")
    ms = C.c_double()
    err = A.photon_err()
    ptr = lambda t: t.data_ptr()  # noqa: E731
    rc = A.lib().photon_debug_layernorm(y_bf16, M, d, ptr(x), ptr(gain), ptr(bias), ptr(y),
                                        ptr(mean), ptr(rstd), ptr(dy), ptr(dres), ptr(dx),
                                        ptr(dxT), ptr(dgain), ptr(dbias), ptr(dsum), C.byref(ms),
                                        C.byref(err))
    assert rc == 0, err.msg
    torch.cuda.synchronize()
    # reference, f64: two-pass mean / var (/n), inv = 1/sqrt(var + 1e-5)
    xd, gd, bd, dyd = x.double(), gain.double(), bias.double(), dy.double()
    mu = xd.mean(1, keepdim=True)
    var = ((xd - mu) ** 2).mean(1, keepdim=True)
    inv = 1.0 / torch.sqrt(var + 1e-5)
    xh = (xd - mu) * inv
    ref_y = gd * xh + bd
    dxh = dyd * gd
    ref_dx = inv * (dxh - dxh.mean(1, keepdim=True) - xh * (dxh * xh).mean(1, keepdim=True))
    ref_out = dres.double() + ref_dx

    def rel(a, b):
        return (a.double() - b).abs().max().item() / (b.abs().max().item() + 1e-30)

    assert rel(mean, mu[:, 0]) <= 1e-5
    assert rel(rstd, inv[:, 0]) <= 1e-5
    assert rel(y, ref_y) <= (8e-3 if y_bf16 else 1e-5)
    assert rel(dx, ref_out) <= 1e-5
    assert rel(dxT, ref_out) <= (8e-3 if y_bf16 else 1e-5)
    assert rel(dgain, (dyd * xh).sum(0)) <= 1e-4
    assert rel(dbias, dyd.sum(0)) <= 1e-4
    assert rel(dsum, ref_out.sum(0)) <= 1e-4


# ---------------------------------------------------------------------------
# GEMMs with a many-band grouped raster
# ---------------------------------------------------------------------------
def _gemm_rows(M, N, K, a_kmajor, b_kmajor, epi, c_bf16, rows, seed=0):
    """Run one tcgen05 GEMM, return (C rows, reference rows) for the sampled rows."""
    A = _A()
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    b = (torch.randn(K, N, device="cuda", generator=g) * 0.05).bfloat16()
    A_st = a if a_kmajor else a.t().contiguous()
    B_st = b.t().contiguous() if b_kmajor else b
    lda = K if a_kmajor else M
    ldb = K if b_kmajor else N
    bias = torch.randn(N, device="cuda", generator=g) * 0.5
    resid = torch.randn(M, N, device="cuda", generator=g) if epi == 3 else None
    cdt = torch.bfloat16 if c_bf16 else torch.float32
    out = torch.zeros(M, N, device="cuda", dtype=cdt)
    aux = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16) if epi == 4 else None
    ms = C.c_double()
    err = A.photon_err()
    rc = A.lib().photon_debug_gemm(1, M, N, K, A_st.data_ptr(), lda, int(a_kmajor),
                                   B_st.data_ptr(), ldb, int(b_kmajor), 1, out.data_ptr(), N,
                                   int(c_bf16), epi, bias.data_ptr(),
                                   resid.data_ptr() if resid is not None else None,
                                   aux.data_ptr() if aux is not None else None, 1, C.byref(ms),
                                   C.byref(err))
    assert rc == 0, err.msg
    torch.cuda.synchronize()
    acc = a[rows].float() @ b.float()
    if epi == 0:
        ref = acc
    elif epi == 2:
        ref = acc + bias
    elif epi == 3:
        ref = resid[rows] + (acc + bias)
    elif epi == 4:
        ref = torch.nn.functional.gelu(acc + bias)
    return out[rows].float(), ref


def _sample_rows(M, tile=256, per_tile=2, seed=0):
    # a few rows of EVERY 256-row tile (so every band and every tile position
    # within a band is checked), plus the first and last rows
    g = torch.Generator().manual_seed(seed)
    n_t = (M + tile - 1) // tile
    r = torch.randint(0, tile, (n_t, per_tile), generator=g) + torch.arange(n_t)[:, None] * tile
    r = torch.cat([r.flatten(), torch.tensor([0, M - 1])]).clamp(max=M - 1)
    return torch.unique(r).cuda()


@pytest.mark.parametrize("M,N,K,epi,c_bf16", [
    (65536, 768, 768, 2, True),     # q / k / v projections (bias epilogue)
    (65536, 3072, 768, 4, True),    # mlp.w1 with the GELU epilogue
    (65536, 768, 3072, 3, False),   # mlp.w2 + residual (fp32 residual stream)
    (16384, V125, 768, 2, True),    # head: 197 column tiles, 64 row tiles (2 bands of 32)
])
def test_gemm_forward_many_bands(M, N, K, epi, c_bf16):
    rows = _sample_rows(M)
    got, ref = _gemm_rows(M, N, K, True, False, epi, c_bf16, rows)
    scale = ref.abs().max().item()
    tol = 1e-2 if c_bf16 else 1e-4
    assert (got - ref).abs().max().item() / scale <= tol


@pytest.mark.parametrize("M,N,K", [(65536, 768, 3072), (16384, 768, V125)])
def test_gemm_dx_many_bands(M, N, K):
    # dX = G W^T: both operands K-major (the weight read in its [in, out] layout)
    rows = _sample_rows(M)
    got, ref = _gemm_rows(M, N, K, True, True, 0, False, rows, seed=1)
    assert (got - ref).abs().max().item() / ref.abs().max().item() <= 1e-4


@pytest.mark.parametrize("M,N,K", [(768, 3072, 65536), (768, V125, 16384)])
def test_gemm_dw_split_k(M, N, K):
    # dW = X^T G: both operands MN-major (no transposed copies), split-K over
    # the token dimension with the deterministic fixed-order reduction
    rows = torch.arange(M, device="cuda")
    got, ref = _gemm_rows(M, N, K, False, False, 0, False, rows, seed=2)
    assert (got - ref).abs().max().item() / ref.abs().max().item() <= 1e-4
