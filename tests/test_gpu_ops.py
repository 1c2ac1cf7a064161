"""GPU parity of each kernel (called through the C ABI) against the oracle.

Tolerance (BASELINE.json north_star, reading R14): per output tensor the
normwise relative error ‖gpu − ref‖₂/‖ref‖₂ ≤ 2e-2 for bf16. The oracle
computes in fp64 from the same bf16 inputs and rounds its outputs to bf16
(R12), so the expected error is ~1e-3; elementwise checks use a bf16-ulp
bound where the arithmetic allows it.
"""
import math

import numpy as np
import pytest

import synth
from oracle import layer as OL
from parity import assert_elementwise

pytestmark = pytest.mark.gpu

TOL = 2e-2


def _torch():
    import torch
    return torch


def dev_bf16(bits):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def host_f64(t):
    torch = _torch()
    if t.dtype == torch.bfloat16:
        return OL.bf16_to_f64(t.view(torch.int16).cpu().numpy().view(np.uint16))
    return t.double().cpu().numpy()


def relerr(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.fixture(scope="module")
def kd(cuda_ok):
    import paper_2604_10180_b200.api as api
    from paper_2604_10180_b200 import _kd
    return api, _kd


def scratch_for(api, op, attrs):
    torch = _torch()
    n = api.op_scratch_bytes(op, attrs)
    return torch.zeros(max(n, 256), dtype=torch.uint8, device="cuda")


# ------------------------------------------------------------------ a3
@pytest.mark.parametrize("rows,H,has_delta", [(1, 256, 0), (5, 4096, 1), (3, 8192, 1), (2, 264, 1)])
def test_add_rmsnorm(kd, rows, H, has_delta):
    api, K = kd
    torch = _torch()
    g = synth.rng(rows * 1000 + H)
    r = synth.normal_f32(g, (rows, H))
    d = synth.normal_bf16(g, (rows, H))
    gam = synth.f32_to_bf16_bits(1 + 0.1 * g.standard_normal(H, dtype=np.float32))
    r_t = torch.from_numpy(r).cuda()
    h_t = torch.empty(rows, H, dtype=torch.bfloat16, device="cuda")
    a = K.kd_attr_add_rmsnorm(rows, H, has_delta, K.KD_BF16, 1e-5, 0)
    api.add_rmsnorm(a, r_t, dev_bf16(d) if has_delta else None, dev_bf16(gam), h_t)
    torch.cuda.synchronize()
    r_ref, h_ref = OL.add_rmsnorm(r, OL.bf16_to_f64(d) if has_delta else None, OL.bf16_to_f64(gam), 1e-5, "bf16")
    assert np.array_equal(host_f64(r_t), r_ref)           # fp32 add is exact-rounded on both sides
    assert relerr(host_f64(h_t), h_ref) < 5e-3
    # elementwise: within 1 bf16 ulp of the oracle's rounded value
    ulp = np.abs(h_ref) * 2.0 ** -7 + 1e-30
    assert np.all(np.abs(host_f64(h_t) - h_ref) <= 1.01 * ulp)


# ------------------------------------------------------------------ GEMM
GEMM_SHAPES = [
    (1, 768, 256),      # tiny QKV, one token
    (4, 256, 1024),     # tiny down
    (33, 384, 320),     # ragged M (mma_n 48), K not a multiple of 128
    (32, 6144, 4096),   # 8B QKV at m=32
    (64, 4096, 4096),   # 8B O at m=64 (split across SMs)
    (32, 4096, 4096),   # 8B O at the disaggregated pair's m=32 (N=2)
    (32, 4096, 14336),  # 8B down at m=32
    (32, 28672, 4096),  # 8B gate_up at m=32
    (96, 6144, 4096),   # the 3:1 role layout's GEMM rows (3 x 32)
    (224, 6144, 4096),  # the 7:1 layout (7 x 32): QKV, O, gate_up, down
    (224, 4096, 4096),
    (224, 28672, 4096),
    (224, 4096, 14336),
    (64, 4096, 14336),  # 8B down (stream-K fixup)
    (64, 28672, 4096),  # 8B gate_up
    (128, 1024, 2048),  # m=128
    (200, 1000, 520),   # two 128-row token blocks, N not a multiple of 16
    (5, 1003, 264),     # odd N (scalar tail stores)
]

@pytest.mark.parametrize("M,N,K_", GEMM_SHAPES)
def test_gemm(kd, M, N, K_):
    """Default tiling per shape (the runtime's choice): every element within
    one bf16 rounding step of the oracle (+1e-3·rms for near-zero sums)."""
    api, K = kd
    torch = _torch()
    g = synth.rng(M * 7 + N * 3 + K_)
    X = synth.normal_bf16(g, (M, K_))
    W = synth.normal_bf16(g, (N, K_), 1 / math.sqrt(K_))
    a = K.kd_attr_gemm(M, N, K_, K.KD_BF16)
    Y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    api.gemm(a, dev_bf16(X), dev_bf16(W), Y, scratch_for(api, K.KD_OP_GEMM, a))
    torch.cuda.synchronize()
    ref = OL.linear(OL.bf16_to_f64(X), OL.bf16_to_f64(W), "bf16")
    assert relerr(host_f64(Y), ref) < 5e-3
    assert_elementwise(host_f64(Y), ref, 1, 1e-3, "gemm Y")


# forced GEMM variants: cluster split-K at a given split (KD_GEMM_TILE, the
# DSMEM reduction in rank order) and stream-K with either fold (KD_GEMM_FOLD:
# last-arriver / grid-wide); all within tolerance and bitwise deterministic
GEMM_TILES = [({"KD_GEMM_TILE": "1"}, 64, 1024, 1024), ({"KD_GEMM_TILE": "2"}, 64, 1024, 1024),
              ({"KD_GEMM_TILE": "3"}, 33, 1024, 1000), ({"KD_GEMM_TILE": "4"}, 64, 4096, 4096),
              ({"KD_GEMM_TILE": "8"}, 100, 1024, 2048), ({"KD_GEMM_TILE": "4"}, 1, 250, 4096),
              ({"KD_GEMM_STREAMK": "1", "KD_GEMM_FOLD": "0"}, 64, 4096, 4096),
              ({"KD_GEMM_STREAMK": "1", "KD_GEMM_FOLD": "1"}, 64, 4096, 4096),
              ({"KD_GEMM_STREAMK": "1", "KD_GEMM_FOLD": "1"}, 48, 28672, 4096)]


@pytest.mark.parametrize("tile,M,N,K_", GEMM_TILES)
def test_gemm_forced_variants(kd, tile, M, N, K_, monkeypatch):
    api, K = kd
    torch = _torch()
    for k, v in tile.items():
        monkeypatch.setenv(k, v)
    g = synth.rng(M * 11 + N * 5 + K_)
    X = synth.normal_bf16(g, (M, K_))
    W = synth.normal_bf16(g, (N, K_), 1 / math.sqrt(K_))
    a = K.kd_attr_gemm(M, N, K_, K.KD_BF16)
    Xd, Wd = dev_bf16(X), dev_bf16(W)
    Y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    scr = scratch_for(api, K.KD_OP_GEMM, a)
    api.gemm(a, Xd, Wd, Y, scr)
    torch.cuda.synchronize()
    Y1 = Y.clone()
    api.gemm(a, Xd, Wd, Y, scr)
    torch.cuda.synchronize()
    assert torch.equal(Y, Y1), "GEMM is not bitwise deterministic"
    ref = OL.linear(OL.bf16_to_f64(X), OL.bf16_to_f64(W), "bf16")
    assert relerr(host_f64(Y), ref) < 5e-3
    assert_elementwise(host_f64(Y), ref, 1, 1e-3, "gemm Y (forced tiling)")


# ------------------------------------------------------------------ a5
@pytest.mark.parametrize("rows,Hq,Hkv,D,C,lens", [(4, 4, 4, 64, 128, None), (3, 32, 8, 128, 4096, None),
                                                  (2, 8, 2, 128, 37, None),
                                                  (6, 32, 8, 128, 4096, [1, 16, 17, 32, 4095, 4096])])
def test_rope_append(kd, rows, Hq, Hkv, D, C, lens):
    api, K = kd
    torch = _torch()
    g = synth.rng(rows + Hq + C)
    theta = 5e5
    qkv = synth.normal_bf16(g, (rows, (Hq + 2 * Hkv) * D))
    pps = (C + 15) // 16
    bt = synth.block_table(g, rows, pps)
    sl = np.full(rows, C, np.int32) if lens is None else np.array(lens, np.int32)  # appends at page ends/starts
    kc = synth.normal_bf16(g, (rows * pps, Hkv, 16, D))
    vc = synth.normal_bf16(g, (rows * pps, Hkv, 16, D))
    kd_, vd_ = dev_bf16(kc), dev_bf16(vc)
    q = torch.empty(rows, Hq * D, dtype=torch.bfloat16, device="cuda")
    a = K.kd_attr_rope_append(rows, Hq, Hkv, D, 16, pps, K.KD_BF16, 0, theta)
    api.rope_append(a, dev_bf16(qkv), torch.from_numpy(bt).cuda(), torch.from_numpy(sl).cuda(), q, kd_, vd_)
    torch.cuda.synchronize()
    kr, vr = OL.bf16_to_f64(kc), OL.bf16_to_f64(vc)
    qr = OL.rope_append(OL.bf16_to_f64(qkv), sl - 1, bt, kr, vr, Hq, Hkv, D, theta, 16, "bf16")
    assert relerr(host_f64(q), qr) < 5e-3
    assert_elementwise(host_f64(q), qr, 1, 1e-4, "rope q")
    kg, vg = host_f64(kd_), host_f64(vd_)
    assert np.array_equal(vg, vr)                       # copy is exact
    assert relerr(kg, kr) < 5e-3
    assert_elementwise(kg, kr, 1, 1e-4, "rope k cache")
    untouched = np.ones(kc.shape[:3], bool)
    for b in range(rows):
        untouched[bt[b][(sl[b] - 1) // 16], :, (sl[b] - 1) % 16] = False
    assert np.array_equal(kg[untouched], OL.bf16_to_f64(kc)[untouched])


# ------------------------------------------------------------------ a6
ATTN = [
    (4, 4, 4, 64, 128),     # tiny (MHA, D=64)
    (2, 32, 8, 128, 4096),  # 8B shape, G=4
    (3, 8, 2, 128, 1000),   # ragged context (partial last page)
    (2, 64, 8, 128, 2048),  # 70B shape, G=8
    (5, 4, 2, 128, 1),      # single key
    (1, 8, 1, 64, 17),      # G=8 MQA, D=64, 2 pages
    (64, 32, 8, 128, 4096), # full 8B bench launch (m=64): 4 splits x 64 pages, 8 ring rounds per CTA
]


@pytest.mark.parametrize("rows,Hq,Hkv,D,C", ATTN)
def test_attention(kd, rows, Hq, Hkv, D, C):
    api, K = kd
    torch = _torch()
    g = synth.rng(rows * 31 + Hq + C)
    pps = (C + 15) // 16
    bt = synth.block_table(g, rows, pps)
    sl = np.full(rows, C, np.int32)
    kc = synth.normal_bf16(g, (rows * pps, Hkv, 16, D))
    vc = synth.normal_bf16(g, (rows * pps, Hkv, 16, D))
    q = synth.normal_bf16(g, (rows, Hq * D))
    out = torch.empty(rows, Hq * D, dtype=torch.bfloat16, device="cuda")
    a = K.kd_attr_attention(rows, Hq, Hkv, D, 16, pps, K.KD_BF16, 0)
    scr = scratch_for(api, K.KD_OP_ATTENTION, a)
    args = (dev_bf16(q), dev_bf16(kc), dev_bf16(vc), torch.from_numpy(bt).cuda(), torch.from_numpy(sl).cuda())
    api.attention(a, *args, out, scr)
    torch.cuda.synchronize()
    o1 = out.clone()
    api.attention(a, *args, out, scr)
    torch.cuda.synchronize()
    assert torch.equal(out, o1), "attention is not bitwise deterministic"
    ref = OL.paged_decode_attention(OL.bf16_to_f64(q), OL.bf16_to_f64(kc), OL.bf16_to_f64(vc), bt, sl, Hq, Hkv, D,
                                    16, "bf16")
    e = relerr(host_f64(out), ref)
    assert e < TOL
    assert e < 1e-2
    # probabilities are rounded to bf16 before the PV MMA (DESIGN.md readings):
    # an absolute term of 1e-2·rms on top of two rounding steps
    assert_elementwise(host_f64(out), ref, 2, 1e-2, "attention out")


# per-row RAGGED context lengths (1, a page end, a page start, C−1, C, ...):
# the default (non-LSE) path, the PDL-early page prefetch and the split
# ranges all depend on each row's own length
ATTN_RAGGED = [
    (8, 32, 8, 128, 4096, [1, 15, 16, 17, 4095, 4096, 2048, 33]),
    (6, 4, 4, 64, 128, [1, 16, 17, 127, 128, 64]),
    (64, 32, 8, 128, 4096, None),   # the bench launch shape with seeded ragged lengths in [1, C]
]


@pytest.mark.parametrize("rows,Hq,Hkv,D,C,lens", ATTN_RAGGED)
def test_attention_ragged_lengths(kd, rows, Hq, Hkv, D, C, lens):
    api, K = kd
    torch = _torch()
    g = synth.rng(rows * 53 + Hq + C)
    pps = (C + 15) // 16
    bt = synth.block_table(g, rows, pps)
    sl = np.array(lens, np.int32) if lens is not None else g.integers(1, C + 1, rows).astype(np.int32)
    kc = synth.normal_bf16(g, (rows * pps, Hkv, 16, D))
    vc = synth.normal_bf16(g, (rows * pps, Hkv, 16, D))
    q = synth.normal_bf16(g, (rows, Hq * D))
    out = torch.empty(rows, Hq * D, dtype=torch.bfloat16, device="cuda")
    a = K.kd_attr_attention(rows, Hq, Hkv, D, 16, pps, K.KD_BF16, 0)
    scr = scratch_for(api, K.KD_OP_ATTENTION, a)
    api.attention(a, dev_bf16(q), dev_bf16(kc), dev_bf16(vc), torch.from_numpy(bt).cuda(),
                  torch.from_numpy(sl).cuda(), out, scr)
    torch.cuda.synchronize()
    ref = OL.paged_decode_attention(OL.bf16_to_f64(q), OL.bf16_to_f64(kc), OL.bf16_to_f64(vc), bt, sl, Hq, Hkv, D,
                                    16, "bf16")
    assert relerr(host_f64(out), ref) < 1e-2
    for b in range(rows):  # per row (a short row's outputs are larger than a long row's: own rms)
        assert relerr(host_f64(out)[b], ref[b]) < 1e-2, f"row {b} (len {sl[b]})"
        assert_elementwise(host_f64(out)[b], ref[b], 2, 1e-2, f"attention out row {b} (len {sl[b]})")


# ------------------------------------------------------------------ a8
@pytest.mark.parametrize("rows,F", [(1, 1024), (7, 14336), (64, 256)])
def test_silu_mul(kd, rows, F):
    api, K = kd
    torch = _torch()
    g = synth.rng(rows + F)
    gu = synth.normal_bf16(g, (rows, 2 * F))
    out = torch.empty(rows, F, dtype=torch.bfloat16, device="cuda")
    api.silu_mul(K.kd_attr_silu_mul(rows, F, K.KD_BF16, 0), dev_bf16(gu), out)
    torch.cuda.synchronize()
    ref = OL.silu_mul_blocked(OL.bf16_to_f64(gu), 64, "bf16")
    assert relerr(host_f64(out), ref) < 5e-3
    assert_elementwise(host_f64(out), ref, 1, 1e-4, "silu_mul")


def test_residual_add(kd):
    api, K = kd
    torch = _torch()
    g = synth.rng(5)
    r = synth.normal_f32(g, (3, 4096))
    d = synth.normal_bf16(g, (3, 4096))
    rt = torch.from_numpy(r).cuda()
    api.residual_add(K.kd_attr_residual_add(3, 4096, 1, 0), rt, dev_bf16(d))
    torch.cuda.synchronize()
    assert np.array_equal(host_f64(rt), OL.residual_add(r, OL.bf16_to_f64(d)))


def test_add_rmsnorm_multi_delta_is_tp_reduction(kd):
    """n_delta = 4: r' = (((r + δ0) + δ1) + δ2) + δ3 in fp32 (index order), the
    reduction half of the fused TP all-reduce (a14)."""
    api, K = kd
    torch = _torch()
    rows, H, n = 5, 4096, 4
    g = synth.rng(77)
    r = synth.normal_f32(g, (rows, H))
    ds = [synth.normal_bf16(g, (rows, H)) for _ in range(n)]
    gam = synth.f32_to_bf16_bits(1 + 0.1 * g.standard_normal(H, dtype=np.float32))
    r_t = torch.from_numpy(r).cuda()
    h_t = torch.empty(rows, H, dtype=torch.bfloat16, device="cuda")
    dts = [dev_bf16(d) for d in ds]
    api.add_rmsnorm(K.kd_attr_add_rmsnorm(rows, H, n, K.KD_BF16, 1e-5, 0), r_t, dts, dev_bf16(gam), h_t)
    torch.cuda.synchronize()
    acc = r.copy()
    for d in ds:                                   # fp32 sequential adds, index order
        acc = (acc + OL.bf16_to_f64(d).astype(np.float32)).astype(np.float32)
    assert np.array_equal(r_t.cpu().numpy(), acc)
    _, h_ref = OL.add_rmsnorm(r, sum(OL.bf16_to_f64(d) for d in ds), OL.bf16_to_f64(gam), 1e-5, "bf16")
    assert relerr(host_f64(h_t), h_ref) < 5e-3
    rr = torch.from_numpy(r).cuda()
    api.residual_add(K.kd_attr_residual_add(rows, H, n, 0), rr, dts)
    torch.cuda.synchronize()
    assert np.array_equal(rr.cpu().numpy(), acc)


# ------------------------------------------------------------------ the fp32 path (R13): 1e-5 vs the oracle
def dev_f32(bits):
    """bf16-valued draws stored fp32 (exact) on the device."""
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(synth.bf16_bits_to_f32(bits))).cuda()


@pytest.mark.parametrize("M,N,K_", [(1, 768, 256), (4, 2048, 1024), (33, 100, 1000)])
def test_gemm_fp32_1e5(kd, M, N, K_):
    api, K = kd
    torch = _torch()
    g = synth.rng(M * 13 + N + K_)
    X = synth.normal_bf16(g, (M, K_))
    W = synth.normal_bf16(g, (N, K_), 1 / math.sqrt(K_))
    a = K.kd_attr_gemm(M, N, K_, K.KD_F32)
    Y = torch.empty(M, N, dtype=torch.float32, device="cuda")
    api.gemm(a, dev_f32(X), dev_f32(W), Y, scratch_for(api, K.KD_OP_GEMM, a))
    torch.cuda.synchronize()
    ref = OL.linear(OL.bf16_to_f64(X), OL.bf16_to_f64(W), "fp32")
    assert relerr(host_f64(Y), ref) < 1e-5
    # fp32 storage: bound each element by 1e-5·rms (fp32 accumulation order only)
    assert np.all(np.abs(host_f64(Y) - ref) <= 1e-5 * np.sqrt(np.mean(ref * ref)) + 2 * np.abs(ref) * 2.0 ** -24)


@pytest.mark.parametrize("rows,Hq,Hkv,D,C", [(4, 4, 4, 64, 128), (3, 8, 2, 128, 37)])
def test_attention_fp32_1e5(kd, rows, Hq, Hkv, D, C):
    api, K = kd
    torch = _torch()
    g = synth.rng(rows * 17 + Hq + C)
    pps = (C + 15) // 16
    bt = synth.block_table(g, rows, pps)
    sl = np.full(rows, C, np.int32)
    kc = synth.normal_bf16(g, (rows * pps, Hkv, 16, D))
    vc = synth.normal_bf16(g, (rows * pps, Hkv, 16, D))
    q = synth.normal_bf16(g, (rows, Hq * D))
    out = torch.empty(rows, Hq * D, dtype=torch.float32, device="cuda")
    a = K.kd_attr_attention(rows, Hq, Hkv, D, 16, pps, K.KD_F32, 0)
    args = (dev_f32(q), dev_f32(kc), dev_f32(vc), torch.from_numpy(bt).cuda(), torch.from_numpy(sl).cuda())
    api.attention(a, *args, out, scratch_for(api, K.KD_OP_ATTENTION, a))
    torch.cuda.synchronize()
    ref = OL.paged_decode_attention(OL.bf16_to_f64(q), OL.bf16_to_f64(kc), OL.bf16_to_f64(vc), bt, sl, Hq, Hkv, D,
                                    16, "fp32")
    assert relerr(host_f64(out), ref) < 1e-5
    assert np.all(np.abs(host_f64(out) - ref) <= 1e-5 * np.sqrt(np.mean(ref * ref)) + 4 * np.abs(ref) * 2.0 ** -24)


# ------------------------------------------------------------------ a9+a8 fused (KD_OP_GEMM_SILU)
@pytest.mark.parametrize("M,F,K_", [(1, 1024, 256), (64, 14336, 4096), (33, 512, 1000)])
def test_gemm_silu_fused_equals_pair(kd, M, F, K_, monkeypatch):
    """Fused gate_up + SiLU·mul: within tolerance of the oracle's a9 → a8, and
    bit-identical to the GPU pair when both GEMMs run the same stream-K split."""
    api, K = kd
    torch = _torch()
    monkeypatch.setenv("KD_GEMM_STREAMK", "1")
    g = synth.rng(M * 5 + F + K_)
    X = synth.normal_bf16(g, (M, K_))
    W = synth.normal_bf16(g, (2 * F, K_), 1 / math.sqrt(K_))
    a = K.kd_attr_gemm(M, 2 * F, K_, K.KD_BF16)
    scr = scratch_for(api, K.KD_OP_GEMM_SILU, a)
    Xd, Wd = dev_bf16(X), dev_bf16(W)
    out = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
    api.gemm_silu(a, Xd, Wd, out, scr)
    gu = torch.empty(M, 2 * F, dtype=torch.bfloat16, device="cuda")
    api.gemm(a, Xd, Wd, gu, scratch_for(api, K.KD_OP_GEMM, a))
    pair = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
    api.silu_mul(K.kd_attr_silu_mul(M, F, K.KD_BF16, 0), gu, pair)
    torch.cuda.synchronize()
    assert torch.equal(out, pair), "fused gate_up+SiLU differs from the GEMM → SiLU pair"
    rows = np.arange(M) if M * F * K_ <= 2 ** 28 else np.array([0, M // 2, M - 1])
    ref = OL.silu_mul_blocked(OL.linear(OL.bf16_to_f64(X[rows]), OL.bf16_to_f64(W), "bf16"), act="bf16")
    assert relerr(host_f64(out)[rows], ref) < 5e-3
    # gate/up sums may round to the neighbouring bf16 value before SiLU: 2 steps
    assert_elementwise(host_f64(out)[rows], ref, 2, 2e-3, "gate_up+silu")


# ------------------------------------------------------------------ a7/a10 + a3 fused (KD_OP_GEMM_RMSNORM)
@pytest.mark.parametrize("M,N,K_,split", [(64, 4096, 4096, None), (64, 4096, 14336, None), (5, 264, 520, "1"),
                                          (33, 384, 320, "2"), (3, 1024, 2048, "4"), (120, 520, 264, "3"),
                                          (64, 4096, 4096, "2")])
def test_gemm_rmsnorm_fused(kd, M, N, K_, split, monkeypatch):
    """O/down GEMM with the residual add + RMSNorm epilogue (per-token Σr²
    completed across the grid after an in-kernel barrier): r bit-identical to
    the GEMM → add_rmsnorm pair at the same cluster split, h within one bf16
    ulp of the pair's (only the Σr² order differs), both within tolerance of
    the oracle, and bitwise reproducible run to run."""
    api, K = kd
    torch = _torch()
    if split:
        monkeypatch.setenv("KD_GEMM_TILE", split)
    g = synth.rng(M * 7 + N + K_)
    X = synth.normal_bf16(g, (M, K_))
    W = synth.normal_bf16(g, (N, K_), 1 / math.sqrt(K_))
    r0 = synth.normal_f32(g, (M, N))
    gam = synth.f32_to_bf16_bits(1 + 0.1 * g.standard_normal(N, dtype=np.float32))
    Xd, Wd, gd = dev_bf16(X), dev_bf16(W), dev_bf16(gam)
    af = K.kd_attr_gemm_rmsnorm(M, N, K_, K.KD_BF16, 1e-5, 0)
    scr = scratch_for(api, K.KD_OP_GEMM_RMSNORM, af)
    outs = []
    for _ in range(2):
        r = torch.from_numpy(r0).cuda()
        h = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        api.gemm_rmsnorm(af, Xd, Wd, r, gd, h, scr)
        outs.append((r, h))
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1]), "not reproducible"
    r, h = outs[0]
    assert not scr[:8].any(), "grid-barrier words must self-reset"
    # the pair
    ag = K.kd_attr_gemm(M, N, K_, K.KD_BF16)
    y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    api.gemm(ag, Xd, Wd, y, scratch_for(api, K.KD_OP_GEMM, ag))
    rp = torch.from_numpy(r0).cuda()
    hp = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    api.add_rmsnorm(K.kd_attr_add_rmsnorm(M, N, 1, K.KD_BF16, 1e-5, 0), rp, y, gd, hp)
    torch.cuda.synchronize()
    hh, hph = host_f64(h), host_f64(hp)
    if split:
        assert torch.equal(r, rp), "fused residual differs from the GEMM → add pair"
        assert np.all(np.abs(hh - hph) <= 1.01 * (np.abs(hph) * 2.0 ** -7) + 1e-30)
    r_ref, h_ref = OL.add_rmsnorm(r0, OL.linear(OL.bf16_to_f64(X), OL.bf16_to_f64(W), "bf16"), OL.bf16_to_f64(gam),
                                  1e-5, "bf16")
    assert relerr(host_f64(r), r_ref) < 1e-3
    assert relerr(hh, h_ref) < 5e-3
    # a GEMM sum rounding to the neighbouring bf16 value moves r' by one ulp of
    # the GEMM output (|Y| ~ rms 1 → 2^-7), which h carries through the norm
    assert_elementwise(hh, h_ref, 2, 1e-2, "gemm_rmsnorm h")


# ------------------------------------------------------------------ a4+a5 fused (KD_OP_QKV_ROPE)
@pytest.mark.parametrize("rows,H,Hq,Hkv,D,C,split", [(4, 256, 4, 4, 64, 128, "2"), (64, 4096, 32, 8, 128, 4096, "2"),
                                                       (3, 512, 8, 2, 128, 37, "4"), (5, 256, 4, 2, 64, 50, "1")])
def test_qkv_rope_fused_equals_pair(kd, rows, H, Hq, Hkv, D, C, split, monkeypatch):
    """QKV GEMM with the RoPE + append epilogue (W rows pair-interleaved per
    head) is bit-identical to the GEMM → rope_append pair at the same cluster
    split, and within tolerance of the oracle."""
    from paper_2604_10180_b200.decoder import pair_interleave_qkv
    api, K = kd
    torch = _torch()
    monkeypatch.setenv("KD_GEMM_TILE", split)
    g = synth.rng(rows * 3 + H + C)
    theta = 5e5
    N = (Hq + 2 * Hkv) * D
    X = synth.normal_bf16(g, (rows, H))
    W = synth.normal_bf16(g, (N, H), 1 / math.sqrt(H))
    pps = (C + 15) // 16
    bt = synth.block_table(g, rows, pps)
    sl = np.full(rows, C, np.int32)
    kc = synth.normal_bf16(g, (rows * pps, Hkv, 16, D))
    vc = synth.normal_bf16(g, (rows * pps, Hkv, 16, D))
    btd, sld = torch.from_numpy(bt).cuda(), torch.from_numpy(sl).cuda()
    # the pair: GEMM then rope_append
    ag = K.kd_attr_gemm(rows, N, H, K.KD_BF16)
    qkv = torch.empty(rows, N, dtype=torch.bfloat16, device="cuda")
    api.gemm(ag, dev_bf16(X), dev_bf16(W), qkv, scratch_for(api, K.KD_OP_GEMM, ag))
    q1, k1, v1 = torch.empty(rows, Hq * D, dtype=torch.bfloat16, device="cuda"), dev_bf16(kc), dev_bf16(vc)
    api.rope_append(K.kd_attr_rope_append(rows, Hq, Hkv, D, 16, pps, K.KD_BF16, 0, theta), qkv, btd, sld, q1, k1, v1)
    # fused
    af = K.kd_attr_qkv_rope(rows, H, Hq, Hkv, D, 16, pps, K.KD_BF16, theta)
    q2, k2, v2 = torch.empty(rows, Hq * D, dtype=torch.bfloat16, device="cuda"), dev_bf16(kc), dev_bf16(vc)
    api.qkv_rope(af, dev_bf16(X), dev_bf16(pair_interleave_qkv(W, D)), btd, sld, q2, k2, v2,
                 scratch_for(api, K.KD_OP_QKV_ROPE, af))
    torch.cuda.synchronize()
    assert torch.equal(q1, q2) and torch.equal(k1, k2) and torch.equal(v1, v2), "fused QKV+RoPE differs from the pair"
    kr, vr = OL.bf16_to_f64(kc), OL.bf16_to_f64(vc)
    qkv_ref = OL.linear(OL.bf16_to_f64(X), OL.bf16_to_f64(W), "bf16")
    qr = OL.rope_append(qkv_ref, sl - 1, bt, kr, vr, Hq, Hkv, D, theta, 16, "bf16")
    assert relerr(host_f64(q2), qr) < 5e-3
    assert relerr(host_f64(k2), kr) < 5e-3 and relerr(host_f64(v2), vr) < 5e-3
    # (a rotation pair mixes two GEMM outputs: one rounding step of either, 2^-7·rms)
    assert_elementwise(host_f64(q2), qr, 2, 1e-2, "qkv_rope q")
    assert_elementwise(host_f64(k2), kr, 2, 1e-2, "qkv_rope k cache")
    assert_elementwise(host_f64(v2), vr, 1, 1e-3, "qkv_rope v cache")


# ------------------------------------------------------------------ f2: attention partials + LSE merge
def test_attention_lse_partials_and_merge(kd):
    api, K = kd
    torch = _torch()
    g = synth.rng(4242)
    rows, Hq, Hkv, D, C, S = 5, 32, 8, 128, 1024, 3
    pps = C // 16
    bt = synth.block_table(g, rows, pps)
    kc = synth.normal_bf16(g, (rows * pps, Hkv, 16, D))
    vc = synth.normal_bf16(g, (rows * pps, Hkv, 16, D))
    q = synth.normal_bf16(g, (rows, Hq * D))
    sl = np.array([1024, 1000, 700, 341, 17], np.int32)  # ragged; some shards empty for some rows
    bounds = [0, 336, 672, 1024]                        # page-aligned, unequal shards
    parts, ref_outs, ref_lses = [], [], []
    for s in range(S):
        p0, p1 = bounds[s] // 16, bounds[s + 1] // 16
        bts = np.ascontiguousarray(bt[:, p0:p1])
        sls = np.clip(sl - bounds[s], 0, bounds[s + 1] - bounds[s]).astype(np.int32)
        a = K.kd_attr_attention(rows, Hq, Hkv, D, 16, p1 - p0, K.KD_BF16, K.KD_ATTN_LSE)
        buf = torch.empty(rows * Hq * D * 2 + rows * Hq * 4, dtype=torch.uint8, device="cuda")
        api.attention(a, dev_bf16(q), dev_bf16(kc), dev_bf16(vc), torch.from_numpy(bts).cuda(),
                      torch.from_numpy(sls).cuda(), buf, scratch_for(api, K.KD_OP_ATTENTION, a))
        parts.append(buf)
        o, l = OL.paged_decode_attention_lse(OL.bf16_to_f64(q), OL.bf16_to_f64(kc), OL.bf16_to_f64(vc), bts, sls,
                                             Hq, Hkv, D)
        ref_outs.append(o)
        ref_lses.append(l)
    torch.cuda.synchronize()
    for s in range(S):
        lse = parts[s][rows * Hq * D * 2:].view(torch.float32).cpu().numpy().reshape(rows, Hq)
        fin = np.isfinite(ref_lses[s])
        assert np.array_equal(np.isfinite(lse), fin)
        assert np.allclose(lse[fin], ref_lses[s][fin], atol=2e-3)
    out = torch.empty(rows, Hq * D, dtype=torch.bfloat16, device="cuda")
    import ctypes as C
    ptrs = (C.c_void_p * S)(*[p.data_ptr() for p in parts])
    K.check(K.kd_op_attn_merge(C.byref(K.kd_attr_attn_merge(rows, Hq, D, S)), ptrs, C.c_void_p(out.data_ptr()),
                               None), "kd_op_attn_merge")
    torch.cuda.synchronize()
    full = OL.paged_decode_attention(OL.bf16_to_f64(q), OL.bf16_to_f64(kc), OL.bf16_to_f64(vc), bt, sl, Hq, Hkv, D,
                                     16, "bf16")
    assert relerr(host_f64(out), OL.lse_merge(ref_outs, ref_lses, D)) < 1e-2
    assert relerr(host_f64(out), full) < 1e-2
    assert_elementwise(host_f64(out), full, 3, 1.5e-2, "merged attention")
