"""Pins for the Mamba-2 (a12) oracle functions: closed forms, special cases
that reduce to textbook expressions, and scalar brute force. CPU only."""
import math

import numpy as np

import synth
from oracle import layer as L


def rs(s):
    return np.random.default_rng(s)


def test_conv_newest_tap_only_is_silu_of_input_and_state_shifts():
    g = rs(1)
    m, Ch, W = 3, 10, 4
    x = g.normal(size=(m, Ch))
    st = g.normal(size=(m, Ch, W - 1))
    w = np.zeros((Ch, W))
    w[:, W - 1] = 1.0
    out, new = L.mamba_conv_step(x, st, w, np.zeros(Ch), act="f64")
    assert np.allclose(out, x / (1 + np.exp(-x)), atol=1e-15)
    assert np.array_equal(new[:, :, :W - 2], st[:, :, 1:]) and np.array_equal(new[:, :, W - 2], x)


def test_conv_bruteforce_loop():
    g = rs(2)
    m, Ch, W = 2, 5, 4
    x, st = g.normal(size=(m, Ch)), g.normal(size=(m, Ch, W - 1))
    w, b = g.normal(size=(Ch, W)), g.normal(size=Ch)
    out, _ = L.mamba_conv_step(x, st, w, b, act="f64")
    for i in range(m):
        for c in range(Ch):
            win = list(st[i, c]) + [x[i, c]]
            pre = sum(win[t] * w[c, t] for t in range(W)) + b[c]
            assert abs(out[i, c] - pre / (1 + math.exp(-pre))) < 1e-12


def _ssm_inputs(seed, m=2, nh=4, P=3, N=5, G=2):
    g = rs(seed)
    return (g.normal(size=(m, nh * P)), g.normal(size=(m, G * N)), g.normal(size=(m, G * N)),
            g.normal(size=(m, nh)), g.normal(size=nh), g.normal(size=nh), g.normal(size=nh),
            g.normal(size=(m, nh, P, N)), nh, P, N, G)


def test_ssm_dt_to_zero_keeps_state():
    x, B, C, dt, dtb, Alog, D, S, nh, P, N, G = _ssm_inputs(3)
    dt = np.full_like(dt, -80.0)
    dtb = np.zeros_like(dtb)
    y, S2 = L.mamba_ssm_step(x, B, C, dt, dtb, Alog, D, S, nh, P, N, G, act="f64")
    assert np.allclose(S2, L.round_f32(S), atol=1e-12)
    hpg = nh // G
    for b in range(2):
        for h in range(nh):
            g = h // hpg
            ref = S[b, h] @ C[b, g * N:(g + 1) * N] + D[h] * x[b, h * P:(h + 1) * P]
            assert np.allclose(y[b, h * P:(h + 1) * P], ref, atol=1e-9)


def test_ssm_instant_decay_is_outer_product_update():
    x, B, C, dt, dtb, Alog, D, S, nh, P, N, G = _ssm_inputs(4)
    Alog = np.full_like(Alog, 60.0)          # A = −e^60: exp(dt·A) underflows to 0
    y, S2 = L.mamba_ssm_step(x, B, C, dt, dtb, Alog, D, S, nh, P, N, G, act="f64")
    hpg = nh // G
    for b in range(2):
        for h in range(nh):
            g = h // hpg
            d = L.softplus(dt[b, h] + dtb[h])
            xs = x[b, h * P:(h + 1) * P]
            Bs, Cs = B[b, g * N:(g + 1) * N], C[b, g * N:(g + 1) * N]
            assert np.allclose(S2[b, h], L.round_f32(d * np.outer(xs, Bs)), atol=1e-12)
            assert np.allclose(y[b, h * P:(h + 1) * P], d * xs * np.dot(Bs, Cs) + D[h] * xs, atol=1e-9)


def test_ssm_scalar_bruteforce():
    x, B, C, dt, dtb, Alog, D, S, nh, P, N, G = _ssm_inputs(5, m=1, nh=2, P=2, N=3, G=1)
    y, S2 = L.mamba_ssm_step(x, B, C, dt, dtb, Alog, D, S, nh, P, N, G, act="f64")
    for h in range(nh):
        d = math.log1p(math.exp(dt[0, h] + dtb[h]))
        dA = math.exp(d * -math.exp(Alog[h]))
        for p in range(P):
            acc = 0.0
            for n in range(N):
                s = S[0, h, p, n] * dA + d * x[0, h * P + p] * B[0, n]
                assert abs(S2[0, h, p, n] - float(np.float32(s))) < 1e-6 * max(1, abs(s))
                acc += s * C[0, n]
            assert abs(y[0, h * P + p] - (acc + D[h] * x[0, h * P + p])) < 1e-12


def test_softplus_matches_definition_and_threshold():
    for v in (-30.0, -1.0, 0.0, 0.7, 19.0, 25.0):
        assert abs(L.softplus(np.array([v]))[0] - (v if v > 20 else math.log1p(math.exp(v)))) < 1e-12


def test_gated_rmsnorm_constant_group_closed_form():
    m, n, gs = 2, 16, 8
    y = np.full((m, n), 0.25)
    z = np.full((m, n), 50.0)               # silu(50) = 50 to double precision
    w = np.ones(n)
    out = L.gated_rmsnorm(y, z, w, gs, 1e-5, act="f64")
    c = 0.25 * 50.0
    assert np.allclose(out, c / math.sqrt(c * c + 1e-5), rtol=1e-12)
    # zero gate → zero output
    assert np.all(L.gated_rmsnorm(y, np.zeros((m, n)), w, gs, 1e-5, act="f64") == 0)


def test_gated_rmsnorm_two_groups_different_scales_hand_value():
    """Pins the GROUPING of the gated RMSNorm (C1.13: groups of d_inner/G
    contiguous channels, each normalised by its own RMS). z = 50 makes
    silu(z) = 50 exactly in fp64. y = [3, 4, 1, 1] with groups of 2:
    group [3, 4] has rms √12.5, group [1, 1] rms 1, so out = [3/√12.5,
    4/√12.5, 1, 1]·w. Row-wise normalisation would give [1.1547, 1.5396,
    0.3849, 0.3849]; interleaved groups ([3, 1], [4, 1]) other values."""
    y = np.array([[3.0, 4.0, 1.0, 1.0]])
    z = np.full((1, 4), 50.0)
    w = np.array([1.0, 2.0, 3.0, 4.0])
    out = L.gated_rmsnorm(y, z, w, 2, 1e-5, act="f64")
    hand = np.array([0.848528137423857, 1.131370849898476 * 2, 1.0 * 3, 1.0 * 4])
    assert np.allclose(out[0], hand, rtol=1e-8, atol=0)  # eps = 1e-5 against ms ≥ 2500: < 2e-9 relative


def test_hybrid_zero_output_projections_pass_residual_and_advance_states():
    cfg = synth.TINY_HYBRID.with_(n_micro=1)
    inp = synth.make_decoder_inputs(cfg)
    for l, lw in enumerate(inp.layers):
        if cfg.is_attn_layer(l):
            lw.w_o = np.zeros_like(lw.w_o)
            lw.w_d = np.zeros_like(lw.w_d)
        else:
            lw.w_out = np.zeros_like(lw.w_out)
    r, convs, ssms = L.hybrid_step(inp, act="fp32")
    assert np.array_equal(r, L.round_f32(inp.x))
    # conv state advanced by one position (oldest dropped)
    l0 = [l for l in range(cfg.n_layers) if not cfg.is_attn_layer(l)][0]
    old = L.bf16_to_f64(inp.conv_state[l0])
    assert np.array_equal(convs[0][:, :, :-1], L.round_f32(old[:, :, 1:]))
