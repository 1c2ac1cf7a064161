"""f4 prefill kernels through the C ABI vs the prefill
oracle (oracle/prefill.py, pinned in test_oracle_prefill.py) and the layer
oracle's GEMM: the large-M tensor-bound GEMM (KD_OP_GEMM with M > 256), RoPE
at every prompt position + paged KV fill, causal GQA attention. Normwise gate
(R14) plus element-wise bounds (parity.py)."""
import numpy as np
import pytest

import synth
from oracle import layer as OL, prefill as PF
from parity import assert_elementwise

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def dev_bf16(bits):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def host_f64(t):
    torch = _torch()
    return OL.bf16_to_f64(t.view(torch.int16).cpu().numpy().view(np.uint16))


def relerr(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-30))


@pytest.fixture(scope="module")
def kd(cuda_ok):
    import paper_2604_10180_b200.api as api
    from paper_2604_10180_b200 import _kd
    return api, _kd


# (M, N, K): several 128x256 tiles per CTA, ragged M / N / K tails, an 8B-shaped QKV at 2K tokens
GEMMS = [(512, 768, 256), (300, 1040, 200), (1024, 512, 1024), (2048, 6144, 4096)]


@pytest.mark.parametrize("M,N,K", GEMMS)
def test_prefill_gemm_vs_oracle(kd, M, N, K):
    api, K_ = kd
    torch = _torch()
    g = synth.rng(M + N + K)
    x = synth.normal_bf16(g, (M, K))
    w = synth.normal_bf16(g, (N, K), 1.0 / np.sqrt(K))
    y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    a = K_.kd_attr_gemm(M, N, K, K_.KD_BF16)
    assert api.op_scratch_bytes(K_.KD_OP_GEMM, a) <= 256      # no split-K scratch on the prefill path
    api.gemm(a, dev_bf16(x), dev_bf16(w), y, torch.zeros(256, dtype=torch.uint8, device="cuda"))
    torch.cuda.synchronize()
    rows = np.arange(M) if M * N <= 2_000_000 else np.unique(np.r_[0, 1, 127, 128, M - 1, synth.rng(1).integers(0, M, 60)])
    ref = OL.linear(OL.bf16_to_f64(x[rows]), OL.bf16_to_f64(w), "bf16")
    got = host_f64(y)[rows]
    assert relerr(got, ref) < 5e-3
    assert_elementwise(got, ref, 1, 2e-3, f"prefill gemm {M}x{N}x{K}")


ROPES = [(2, 64, 4, 4, 64, 1e4), (3, 48, 32, 8, 128, 5e5)]


@pytest.mark.parametrize("B,S,Hq,Hkv,D,theta", ROPES)
def test_rope_prefill_vs_oracle(kd, B, S, Hq, Hkv, D, theta):
    api, K_ = kd
    torch = _torch()
    g = synth.rng(B * S + D)
    rows = B * S
    pps = (S + 16 + 15) // 16           # capacity beyond the prompt: untouched slots stay as they were
    qkv = synth.normal_bf16(g, (rows, (Hq + 2 * Hkv) * D))
    bt = synth.block_table(g, B, pps)
    kc = synth.normal_bf16(g, (B * pps, Hkv, 16, D))
    vc = synth.normal_bf16(g, (B * pps, Hkv, 16, D))
    kd_, vd_ = dev_bf16(kc), dev_bf16(vc)
    q = torch.empty(rows, Hq * D, dtype=torch.bfloat16, device="cuda")
    a = K_.kd_attr_rope_prefill(B, S, Hq, Hkv, D, 16, pps, K_.KD_BF16, theta)
    api.rope_prefill(a, dev_bf16(qkv), torch.from_numpy(bt).cuda(), q, kd_, vd_)
    torch.cuda.synchronize()
    kr, vr = OL.bf16_to_f64(kc), OL.bf16_to_f64(vc)
    qr = PF.rope_prefill(OL.bf16_to_f64(qkv), S, bt, kr, vr, Hq, Hkv, D, theta, 16, "bf16")
    assert_elementwise(host_f64(q), qr, 1, 1e-4, "prefill q")
    assert_elementwise(host_f64(kd_), kr, 1, 1e-4, "prefill k cache (incl. untouched slots)")
    assert np.array_equal(host_f64(vd_), vr)                 # v is a copy


ATTN = [(2, 64, 4, 4, 64), (1, 128, 8, 2, 128), (2, 192, 32, 8, 128), (1, 80, 4, 1, 64), (1, 1024, 32, 8, 128)]


@pytest.mark.parametrize("B,S,Hq,Hkv,D", ATTN)
def test_prefill_attention_vs_oracle(kd, B, S, Hq, Hkv, D):
    """Tiles of 64 queries: S = 80 ends in a partial key block (zero-filled V
    rows past the prompt); 1024 = the bench prompt length."""
    api, K_ = kd
    torch = _torch()
    g = synth.rng(B * S + Hq)
    pps = (S + 15) // 16
    bt = synth.block_table(g, B, pps)
    kc = synth.normal_bf16(g, (B * pps, Hkv, 16, D))
    vc = synth.normal_bf16(g, (B * pps, Hkv, 16, D))
    q = synth.normal_bf16(g, (B * S, Hq * D))
    out = torch.empty(B * S, Hq * D, dtype=torch.bfloat16, device="cuda")
    a = K_.kd_attr_prefill_attention(B, S, Hq, Hkv, D, 16, pps, K_.KD_BF16)
    api.prefill_attention(a, dev_bf16(q), dev_bf16(kc), dev_bf16(vc), torch.from_numpy(bt).cuda(), out)
    torch.cuda.synchronize()
    got = host_f64(out)
    ref = PF.prefill_attention(OL.bf16_to_f64(q), OL.bf16_to_f64(kc), OL.bf16_to_f64(vc), bt, S, Hq, Hkv, D, 16, "bf16")
    assert relerr(got, ref) < 1e-2
    # P is rounded to bf16 before P·V (as FlashAttention and the decode kernel
    # do): each term carries a 2^-9 relative error, so a query with few keys
    # (early tokens: out is the average of a handful of |v| ~ 1 values) is off
    # by ~2^-9·|v| whatever |out| is — 2 bf16 ulps at rms scale
    assert_elementwise(got, ref, 2, 2e-2, f"prefill attention B{B} S{S} H{Hq}/{Hkv} D{D}")


def test_prefill_ops_reject_bad_shapes(kd):
    api, K_ = kd
    bad = K_.kd_attr_prefill_attention(1, 40, 4, 4, 96, 16, 3, K_.KD_BF16)  # head_dim 96
    with pytest.raises(K_.KdError):
        api.prefill_attention(bad, None, None, None, None, None)
    bad = K_.kd_attr_prefill_attention(1, 40, 4, 4, 64, 16, 3, K_.KD_BF16)  # seq_len % 16
    with pytest.raises(K_.KdError):
        api.prefill_attention(bad, None, None, None, None, None)
