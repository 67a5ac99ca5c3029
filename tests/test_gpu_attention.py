"""Fused causal attention (tensor-core and SIMT paths) vs a plain PyTorch fp32
reference of the same op (tensor.cpp:436-542 semantics: scale before the max,
keys j <= i).  bf16 inputs/outputs, fp32 math: outputs within 2e-2 of the
output scale, lse within 1e-3 absolute."""
import ctypes as C
import math

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _ref(q, k, v, dO, H):
    B, S, d = q.shape
    dh = d // H
    qf, kf, vf = (x.float().view(B, S, H, dh).transpose(1, 2).requires_grad_(True)
                  for x in (q, k, v))
    s = qf @ kf.transpose(-1, -2) / math.sqrt(dh)
    mask = torch.ones(S, S, device=q.device, dtype=torch.bool).triu(1)
    s = s.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(s, dim=-1)
    p = torch.softmax(s, dim=-1)
    o = p @ vf
    o.backward(dO.float().view(B, S, H, dh).transpose(1, 2))
    back = lambda t: t.transpose(1, 2).reshape(B, S, d)  # noqa: E731
    return back(o.detach()), lse.detach().reshape(B * H * S), back(qf.grad), back(kf.grad), \
        back(vf.grad)


def _run(impl, B, S, H, d, seed=0):
    from paper_2411_02908_b200 import _capi as A

    g = torch.Generator(device="cuda").manual_seed(seed)
    mk = lambda: (torch.randn(B, S, d, device="cuda", generator=g)).bfloat16()  # noqa: E731
    q, k, v, dO = mk(), mk(), mk(), mk()
    o = torch.empty_like(q)
    lse = torch.empty(B * H * S, device="cuda")
    scratch = torch.empty(B * H * S, device="cuda")
    dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
    err = A.photon_err()
    ms_f, ms_b = C.c_double(), C.c_double()
    rc = A.lib().photon_debug_attention(impl, B, S, H, d, q.data_ptr(), k.data_ptr(),
                                        v.data_ptr(), o.data_ptr(), lse.data_ptr(), None, None,
                                        None, None, None, C.byref(ms_f), C.byref(err))
    assert rc == 0, err.msg
    rc = A.lib().photon_debug_attention(impl, B, S, H, d, q.data_ptr(), k.data_ptr(),
                                        v.data_ptr(), o.data_ptr(), lse.data_ptr(), dO.data_ptr(),
                                        scratch.data_ptr(), dq.data_ptr(), dk.data_ptr(),
                                        dv.data_ptr(), C.byref(ms_b), C.byref(err))
    assert rc == 0, err.msg
    torch.cuda.synchronize()
    o_r, lse_r, dq_r, dk_r, dv_r = _ref(q, k, v, dO, H)
    for name, got, want in (("o", o, o_r), ("dq", dq, dq_r), ("dk", dk, dk_r), ("dv", dv, dv_r)):
        rel = (got.float() - want).abs().max().item() / (want.abs().max().item() + 1e-6)
        assert rel <= 2e-2, (name, impl, B, S, H, d, rel)
    assert (lse - lse_r).abs().max().item() <= 1e-3
    return ms_f.value, ms_b.value


@pytest.mark.parametrize("impl", [1, 0])
@pytest.mark.parametrize("B,S,H,d", [(2, 16, 2, 32), (2, 32, 2, 64), (1, 128, 2, 128),
                                     (1, 200, 3, 192), (2, 256, 4, 512)])
def test_attention_small(impl, B, S, H, d):
    _run(impl, B, S, H, d)


def test_attention_photon125m_head_shape():
    # dh = 64, S = 2048 (the 125M shape), tensor-core paths
    _run(1, 2, 2048, 2, 128)
    _run(2, 2, 2048, 2, 128)


@pytest.mark.parametrize("dh", [64, 128])
@pytest.mark.parametrize("B,S,H", [(2, 128, 2), (1, 256, 3), (2, 200, 2), (1, 64, 1), (3, 384, 2),
                                   (1, 320, 1)])
def test_attention_tcgen05(B, S, H, dh):
    # forward + backward on tcgen05 (head dims 64 and 128; the 1.3B / 7B heads are 128)
    _run(2, B, S, H, dh * H)


def test_attention_tcgen05_dh128_long():
    _run(2, 1, 2048, 2, 256)


def test_attention_tcgen05_many_heads():
    # B * H = 192 > 148: the fused dh-64 backward runs on 148 CTAs with heads cut
    # between neighbouring CTAs at key-tile boundaries; odd heads walk their key
    # tiles in descending order
    _run(2, 16, 256, 12, 768)
    _run(2, 16, 640, 12, 768)
    _run(2, 25, 128, 12, 768)   # 300 heads of one key tile each (no cuts possible)
    _run(2, 5, 1000, 30, 1920)  # 150 heads on 148 CTAs: nearly every CTA boundary cuts a head


def test_attention_tcgen05_cut_heads_bitwise():
    # heads cut between two CTAs (B * H = 192 on 148 SMs) give bit-identical dq /
    # dk / dv to the same heads run whole (one sequence per launch: 12 heads,
    # no cuts; H even keeps every head's walking direction)
    from paper_2411_02908_b200 import _capi as A

    B, S, H = 16, 640, 12
    d = 64 * H
    g = torch.Generator(device="cuda").manual_seed(5)
    q, k, v, dO = (torch.randn(B, S, d, device="cuda", generator=g).bfloat16() for _ in range(4))
    err = A.photon_err()
    ms = C.c_double()

    def run(Bn, qq, kk, vv, dd):
        o = torch.empty_like(qq)
        lse = torch.empty(Bn * H * S, device="cuda")
        assert A.lib().photon_debug_attention(2, Bn, S, H, d, qq.data_ptr(), kk.data_ptr(),
                                              vv.data_ptr(), o.data_ptr(), lse.data_ptr(), None,
                                              None, None, None, None, C.byref(ms),
                                              C.byref(err)) == 0, err.msg
        dq, dk, dv = torch.empty_like(qq), torch.empty_like(qq), torch.empty_like(qq)
        assert A.lib().photon_debug_attention(2, Bn, S, H, d, qq.data_ptr(), kk.data_ptr(),
                                              vv.data_ptr(), o.data_ptr(), lse.data_ptr(),
                                              dd.data_ptr(), None, dq.data_ptr(), dk.data_ptr(),
                                              dv.data_ptr(), C.byref(ms), C.byref(err)) == 0, err.msg
        torch.cuda.synchronize()
        return dq, dk, dv

    full = run(B, q, k, v, dO)
    for b in range(B):
        one = run(1, *(x[b:b + 1].contiguous() for x in (q, k, v, dO)))
        for name, x, y in zip(("dq", "dk", "dv"), full, one):
            assert torch.equal(x[b:b + 1], y), (name, b)


def test_attention_tcgen05_backward_deterministic():
    # the fused backward adds dQ partial sums in a fixed key-tile order: two runs
    # are bit-identical, and the result does not depend on CTA scheduling
    from paper_2411_02908_b200 import _capi as A

    B, S, H = 2, 1000, 3
    d = 64 * H
    g = torch.Generator(device="cuda").manual_seed(3)
    q, k, v, dO = (torch.randn(B, S, d, device="cuda", generator=g).bfloat16() for _ in range(4))
    o = torch.empty_like(q)
    lse = torch.empty(B * H * S, device="cuda")
    err = A.photon_err()
    ms = C.c_double()
    assert A.lib().photon_debug_attention(2, B, S, H, d, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                          o.data_ptr(), lse.data_ptr(), None, None, None, None,
                                          None, C.byref(ms), C.byref(err)) == 0, err.msg
    outs = []
    for _ in range(3):
        dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
        assert A.lib().photon_debug_attention(2, B, S, H, d, q.data_ptr(), k.data_ptr(),
                                              v.data_ptr(), o.data_ptr(), lse.data_ptr(),
                                              dO.data_ptr(), None, dq.data_ptr(), dk.data_ptr(),
                                              dv.data_ptr(), C.byref(ms), C.byref(err)) == 0, err.msg
        outs.append((dq, dk, dv))
    for x, y in zip(outs[0], outs[1]):
        assert torch.equal(x, y)
    for x, y in zip(outs[0], outs[2]):
        assert torch.equal(x, y)
