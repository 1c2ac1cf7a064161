"""Pins for oracle/layer.py against closed forms, invariants and brute force
(SURVEY §8(c) "What pins each part", layer math row). CPU only."""
import math

import numpy as np
import pytest

from oracle import layer as L
import synth


def rs(seed=0):
    return np.random.default_rng(seed)


# ------------------------------------------------------------------ storage
def test_bf16_round_known_values():
    # 1 + 2^-8 is exactly halfway between bf16 neighbours 1 and 1+2^-7 -> even (1)
    assert L.round_bf16(np.array([1.0 + 2 ** -8]))[0] == 1.0
    assert L.round_bf16(np.array([1.0 + 3 * 2 ** -9]))[0] == 1.0 + 2 ** -7
    assert L.round_bf16(np.array([-2.0]))[0] == -2.0
    # decode of the encoder in synth is exact for representable values
    x = np.array([1.5, -0.15625, 3.0], np.float32)
    assert np.all(L.bf16_to_f64(synth.f32_to_bf16_bits(x)) == x)


# ------------------------------------------------------------------ a3
def test_rmsnorm_constant_row_closed_form():
    # RMSNorm of c·1 with gamma = 1 -> c / sqrt(c^2 + eps) in every element
    for c in (0.5, -3.0, 2.0 ** -10):  # fp32-representable (residual is stored fp32)
        r = np.full((1, 64), c)
        _, h = L.add_rmsnorm(r, None, np.ones(64), 1e-5, act="f64")
        assert np.allclose(h, c / math.sqrt(c * c + 1e-5), rtol=1e-12)


def test_rmsnorm_add_and_bruteforce_loop():
    g = rs(1)
    r, d, gam = g.normal(size=(3, 32)), g.normal(size=(3, 32)), g.normal(size=32)
    rn, h = L.add_rmsnorm(r, d, gam, 1e-5, act="f64")
    for b in range(3):
        s = [float(np.float32(r[b, j] + d[b, j])) for j in range(32)]
        assert np.allclose(rn[b], s, rtol=0, atol=0)
        ms = sum(v * v for v in s) / 32
        for j in range(32):
            assert abs(h[b, j] - s[j] / math.sqrt(ms + 1e-5) * gam[j]) < 1e-12


def test_rmsnorm_scale_invariance():
    g = rs(2)
    r = g.normal(size=(2, 128))
    _, h1 = L.add_rmsnorm(r, None, np.ones(128), 0.0, act="f64")
    _, h2 = L.add_rmsnorm(7.0 * r, None, np.ones(128), 0.0, act="f64")
    assert np.allclose(h1, h2, rtol=1e-6)  # 7r is rounded to fp32 storage first


# ------------------------------------------------------------------ GEMM
def test_linear_identity_and_triple_loop():
    g = rs(3)
    x = g.normal(size=(3, 8))
    assert np.allclose(L.linear(x, np.eye(8), act="f64"), x)
    W = g.normal(size=(5, 8))
    y = L.linear(x, W, act="f64")
    for i in range(3):
        for n in range(5):
            assert abs(y[i, n] - sum(x[i, k] * W[n, k] for k in range(8))) < 1e-12


# ------------------------------------------------------------------ a5 RoPE
def test_rope_pos0_identity():
    x = rs(4).normal(size=64)
    assert np.allclose(L.rope_neox(x, 0, 1e4), x, rtol=0, atol=0)


def test_rope_d2_is_rotation_by_pos_radians():
    # D = 2: theta^(0) = 1, so the pair rotates by exactly pos radians
    x = np.array([0.3, -1.2])
    for p in (1, 5, 17):
        y = L.rope_neox(x, p, 12345.0)
        c, s = math.cos(p), math.sin(p)
        assert np.allclose(y, [x[0] * c - x[1] * s, x[1] * c + x[0] * s], atol=1e-14)


def test_rope_relative_position_property():
    g = rs(5)
    q, k = g.normal(size=128), g.normal(size=128)
    a = np.dot(L.rope_neox(q, 100, 5e5), L.rope_neox(k, 90, 5e5))
    b = np.dot(L.rope_neox(q, 1010, 5e5), L.rope_neox(k, 1000, 5e5))
    assert abs(a - b) < 1e-9
    assert abs(np.linalg.norm(L.rope_neox(q, 77, 5e5)) - np.linalg.norm(q)) < 1e-12


def test_rope_pairs_halves_not_adjacent():
    # NeoX style pairs i with i + D/2: a vector supported on dim 0 moves to dim D/2
    x = np.zeros(8)
    x[0] = 1.0
    y = L.rope_neox(x, 1, 1e4)
    assert abs(y[0] - math.cos(1)) < 1e-14 and abs(y[4] - math.sin(1)) < 1e-14
    assert np.all(y[[1, 2, 3, 5, 6, 7]] == 0)


def test_rope_frequency_exponent_second_pair_hand_value():
    """Pins θ^(−2i/D) for i ≥ 1 (R12; the Llama/NeoX RoPE frequency
    schedule): D = 4, θ = 10⁴, pos = 3 → pair 0 turns by 3 rad, pair 1 by
    3·10⁴^(−2/4) = 3·10⁻² rad. Hand values (cos 0.03, sin 0.03, cos 3, sin 3)
    are literals, not recomputed from the oracle's formula; a wrong exponent
    (θ^(−i/D), θ^(−2i/(D−2)), θ^(+…)) or swapped pairing fails here."""
    c0, s0 = L.rope_freqs(3, 4, 1e4)
    assert abs(c0[0] - (-0.9899924966004454)) < 1e-15 and abs(s0[0] - 0.1411200080598672) < 1e-15
    assert abs(c0[1] - 0.9995500337489875) < 1e-15 and abs(s0[1] - 0.029995500202495664) < 1e-15
    # a unit vector on the second pair's first half: (0, 1, 0, 0) -> (0, cos .03, 0, sin .03)
    y = L.rope_neox(np.array([0.0, 1.0, 0.0, 0.0]), 3, 1e4)
    assert np.allclose(y, [0.0, 0.9995500337489875, 0.0, 0.029995500202495664], rtol=0, atol=1e-15)
    # D = 8, θ = 10⁴, pos = 1: angles 1, 10⁻¹, 10⁻², 10⁻³ rad (exactly θ^(−2i/8) = 10^(−i))
    c, s = L.rope_freqs(1, 8, 1e4)
    hand_c = [0.5403023058681398, 0.9950041652780258, 0.9999500004166653, 0.9999995000000417]
    hand_s = [0.8414709848078965, 0.09983341664682815, 0.009999833334166664, 0.0009999998333333417]
    assert np.allclose(c, hand_c, rtol=0, atol=1e-15) and np.allclose(s, hand_s, rtol=0, atol=1e-15)


def test_kv_append_slot_and_grouped_split():
    Hq, Hkv, D, P = 4, 2, 4, 16
    G = Hq // Hkv
    qkv = np.arange((Hq + 2 * Hkv) * D, dtype=np.float64)[None, :]
    q, k, v = L.split_qkv_grouped(qkv[0], Hq, Hkv, D)
    # group 1 starts after group 0's (G + 2) * D columns
    assert np.all(k[1] == np.arange((G + 2) * D + G * D, (G + 2) * D + (G + 1) * D))
    assert np.all(q[3] == np.arange((G + 2) * D + D, (G + 2) * D + 2 * D))
    kc = np.zeros((5, Hkv, P, D))
    vc = np.zeros((5, Hkv, P, D))
    bt = np.array([[3, 1]])   # position 17 -> logical page 1 -> physical page 1, slot 1
    L.rope_append(qkv, np.array([17]), bt, kc, vc, Hq, Hkv, D, 1e4, P, act="f64")
    assert np.all(vc[1, :, 1, :] == v)
    assert np.count_nonzero(vc) == np.count_nonzero(v)
    assert np.allclose(kc[1, 0, 1], L.rope_neox(k[0], 17, 1e4))


# ------------------------------------------------------------------ a6 attention
def _one_seq_cache(K, V, P=16):
    C, Hkv, D = K.shape
    npg = (C + P - 1) // P
    kc = np.zeros((npg, Hkv, P, D))
    vc = np.zeros((npg, Hkv, P, D))
    perm = np.arange(npg)[::-1].copy()   # fragmented: logical page j -> physical npg-1-j
    for t in range(C):
        kc[perm[t // P], :, t % P] = K[t]
        vc[perm[t // P], :, t % P] = V[t]
    return kc, vc, perm[None, :]


def test_attention_single_key_returns_v0():
    g = rs(6)
    K, V = g.normal(size=(1, 2, 8)), g.normal(size=(1, 2, 8))
    kc, vc, bt = _one_seq_cache(K, V)
    q = g.normal(size=(1, 4 * 8))
    out = L.paged_decode_attention(q, kc, vc, bt, [1], 4, 2, 8, act="f64")
    for h in range(4):
        assert np.allclose(out[0, h * 8:(h + 1) * 8], V[0, h // 2])


def test_attention_identical_keys_is_mean_of_v():
    g = rs(7)
    C = 37
    K = np.tile(g.normal(size=(1, 1, 16)), (C, 1, 1))
    V = g.normal(size=(C, 1, 16))
    kc, vc, bt = _one_seq_cache(K, V)
    out = L.paged_decode_attention(g.normal(size=(1, 16)), kc, vc, bt, [C], 1, 1, 16, act="f64")
    assert np.allclose(out[0], V[:, 0].mean(axis=0), atol=1e-12)


def test_attention_dominating_score_selects_v():
    g = rs(8)
    C, D = 40, 16
    K = g.normal(size=(C, 1, D)) * 0.01
    K[23, 0] = 50.0 * np.ones(D)
    V = g.normal(size=(C, 1, D))
    kc, vc, bt = _one_seq_cache(K, V)
    out = L.paged_decode_attention(np.ones((1, D)), kc, vc, bt, [C], 1, 1, D, act="f64")
    assert np.allclose(out[0], V[23, 0], atol=1e-9)


def test_attention_matches_materialised_textbook_gqa():
    g = rs(9)
    C, Hq, Hkv, D = 45, 8, 2, 8
    K, V = g.normal(size=(C, Hkv, D)), g.normal(size=(C, Hkv, D))
    kc, vc, bt = _one_seq_cache(K, V)
    q = g.normal(size=(1, Hq * D))
    out = L.paged_decode_attention(q, kc, vc, bt, [C], Hq, Hkv, D, act="f64")
    for h in range(Hq):
        kvh = h // (Hq // Hkv)
        scores = [sum(q[0, h * D + d] * K[t, kvh, d] for d in range(D)) / math.sqrt(D) for t in range(C)]
        mx = max(scores)
        e = [math.exp(s - mx) for s in scores]
        z = sum(e)
        ref = [sum(e[t] / z * V[t, kvh, d] for t in range(C)) for d in range(D)]
        assert np.allclose(out[0, h * D:(h + 1) * D], ref, atol=1e-12)


def test_attention_length_masks_tail():
    g = rs(10)
    C, D = 33, 8
    K, V = g.normal(size=(48, 1, D)), g.normal(size=(48, 1, D))
    kc, vc, bt = _one_seq_cache(K, V)
    q = g.normal(size=(1, D))
    a = L.paged_decode_attention(q, kc, vc, bt, [C], 1, 1, D, act="f64")
    kc2, vc2 = kc.copy(), vc.copy()
    kc2[bt[0, 2], 0, 1:] = 99.0   # positions >= 33 on logical page 2
    vc2[bt[0, 2], 0, 1:] = 99.0
    b = L.paged_decode_attention(q, kc2, vc2, bt, [C], 1, 1, D, act="f64")
    assert np.array_equal(a, b)


# ------------------------------------------------------------------ a8
def test_silu_values_and_block_interleave():
    assert L.silu(np.array([0.0]))[0] == 0.0
    assert abs(L.silu(np.array([1.0]))[0] - 1.0 / (1.0 + math.exp(-1.0))) < 1e-15
    B = 4
    gate = np.array([[0.0, 1.0, -1.0, 2.0, 0.5, 0.5, 0.5, 0.5]])
    up = np.array([[1.0, 1.0, 1.0, 1.0, 2.0, 2.0, 2.0, 2.0]])
    gu = np.concatenate([gate[:, :4], up[:, :4], gate[:, 4:], up[:, 4:]], axis=1)
    a = L.silu_mul_blocked(gu, block=B, act="f64")
    assert np.allclose(a, L.silu(gate) * up)


# ------------------------------------------------------------------ MoE
def test_moe_one_hot_logits_pick_that_expert():
    H, E = 8, 4
    w_r = np.zeros((E, H))
    w_r[2, 0] = 10.0
    w_r[1, 1] = 5.0
    h = np.zeros((1, H))
    h[0, 0] = 1.0
    h[0, 1] = 1.0
    idx, w = L.moe_route(h, w_r, 2)
    assert idx.tolist() == [[2, 1]]
    assert abs(w[0, 0] - 1.0 / (1.0 + math.exp(-5.0))) < 1e-12
    # ties resolve to the lower expert index
    idx, _ = L.moe_route(np.zeros((1, H)), w_r, 2)
    assert idx.tolist() == [[0, 1]]


def test_moe_equals_dense_masked_reference():
    g = rs(11)
    m, H, F, E = 3, 8, 128, 4
    h = g.normal(size=(m, H))
    wr = g.normal(size=(E, H))
    wgu = g.normal(size=(E, 2 * F, H)) * 0.3
    wd = g.normal(size=(E, H, F)) * 0.3
    idx, w = L.moe_route(h, wr, 2)
    out = L.moe_ffn(h, idx, w, wgu, wd, act="f64")
    # dense-with-masks textbook form: every expert on every row, masked weights
    dense = np.zeros((m, H))
    for e in range(E):
        gu = h @ wgu[e].T
        gate = np.concatenate([gu[:, 2 * j * 64: 2 * j * 64 + 64] for j in range(F // 64)], 1)
        up = np.concatenate([gu[:, 2 * j * 64 + 64: 2 * j * 64 + 128] for j in range(F // 64)], 1)
        y = (gate / (1 + np.exp(-gate)) * up) @ wd[e].T
        mask = np.array([w[b][list(idx[b]).index(e)] if e in idx[b] else 0.0 for b in range(m)])
        dense += mask[:, None] * y
    assert np.allclose(out, dense, atol=1e-10)


# ------------------------------------------------------------------ layer
def test_layer_zero_output_projections_pass_residual_through():
    cfg = synth.TINY.with_(n_layers=1, batch=2, context=20, n_micro=1)
    inp = synth.make_decoder_inputs(cfg)
    lw = inp.layers[0]
    lw.w_o = np.zeros_like(lw.w_o)
    lw.w_d = np.zeros_like(lw.w_d)
    r_out, _, _ = L.decoder_step(inp, act="fp32")
    assert np.array_equal(r_out, L.round_f32(inp.x))


def test_layer_composition_matches_unpaged_dense_reference():
    """Whole layer vs an independent dense restatement: contiguous (unpaged)
    KV, natural (non-interleaved) weight order, materialised softmax."""
    cfg = synth.TINY.with_(n_layers=1, batch=2, context=24, n_kv_heads=2, n_micro=2)
    inp = synth.make_decoder_inputs(cfg)
    r_out, _, _ = L.decoder_step(inp, act="f64")
    H, Hq, Hkv, D, F = cfg.hidden, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.ffn
    G = Hq // Hkv
    dec = L.bf16_to_f64
    lw = inp.layers[0]
    Wqkv = dec(lw.w_qkv).reshape(Hkv, G + 2, D, H)
    Wq = Wqkv[:, :G].reshape(Hq * D, H)
    Wk = Wqkv[:, G].reshape(Hkv * D, H)
    Wv = Wqkv[:, G + 1].reshape(Hkv * D, H)
    Wgu = dec(lw.w_gu).reshape(F // 64, 2, 64, H)
    Wg, Wu = Wgu[:, 0].reshape(F, H), Wgu[:, 1].reshape(F, H)
    x = inp.x.astype(np.float64)
    pos = cfg.context - 1
    for b in range(cfg.batch):
        r = np.float32(x[b]).astype(np.float64)
        h = r / np.sqrt(np.mean(r * r) + cfg.eps) * dec(lw.gamma1)
        q, k, v = Wq @ h, Wk @ h, Wv @ h
        Kc = np.stack([dec(inp.k_cache[0][inp.block_table[b][t // 16], :, t % 16]) for t in range(cfg.context)])
        Vc = np.stack([dec(inp.v_cache[0][inp.block_table[b][t // 16], :, t % 16]) for t in range(cfg.context)])
        attn = np.zeros(Hq * D)
        for g in range(Hkv):
            Kc[pos, g] = L.rope_neox(k[g * D:(g + 1) * D], pos, cfg.rope_theta)
            Vc[pos, g] = v[g * D:(g + 1) * D]
        for hh in range(Hq):
            g = hh // G
            qr = L.rope_neox(q[hh * D:(hh + 1) * D], pos, cfg.rope_theta)
            s = Kc[:, g] @ qr / math.sqrt(D)
            p = np.exp(s - s.max())
            p /= p.sum()
            attn[hh * D:(hh + 1) * D] = p @ Vc[:, g]
        r2 = np.float32(r + dec(lw.w_o) @ attn).astype(np.float64)
        h2 = r2 / np.sqrt(np.mean(r2 * r2) + cfg.eps) * dec(lw.gamma2)
        gg, uu = Wg @ h2, Wu @ h2
        d = dec(lw.w_d) @ (gg / (1 + np.exp(-gg)) * uu)
        ref = np.float32(r2 + d).astype(np.float64)
        assert np.allclose(r_out[b], ref, rtol=1e-6, atol=1e-6)


# ------------------------------------------------------------------ f2: KV shards + LSE merge
def test_lse_merge_of_shards_equals_full_attention():
    from oracle import layer as OL
    """Splitting every sequence's keys into disjoint shards and merging the
    shard partials by their log-sum-exp is the softmax over the union (exact
    in fp64), including a shard that holds no key of a sequence."""
    import synth
    g = synth.rng(77)
    m, Hq, Hkv, D, C, S = 3, 4, 2, 32, 48, 3
    pps = C // 16
    bt = synth.block_table(g, m, pps)
    kc = OL.bf16_to_f64(synth.normal_bf16(g, (m * pps, Hkv, 16, D)))
    vc = OL.bf16_to_f64(synth.normal_bf16(g, (m * pps, Hkv, 16, D)))
    q = OL.bf16_to_f64(synth.normal_bf16(g, (m, Hq * D)))
    sl = np.array([48, 20, 33], np.int32)           # sequence 1 has no key in shard 2
    full = OL.paged_decode_attention(q, kc, vc, bt, sl, Hq, Hkv, D, 16, "f64")
    T = C // S
    outs, lses = [], []
    for s in range(S):
        bts = bt[:, s * T // 16:(s + 1) * T // 16]
        sls = np.clip(sl - s * T, 0, T)
        o, l = OL.paged_decode_attention_lse(q, kc, vc, bts, sls, Hq, Hkv, D)
        outs.append(o)
        lses.append(l)
    assert np.isneginf(lses[2][1]).all()
    merged = OL.lse_merge(outs, lses, D)
    assert np.allclose(merged, full, rtol=0, atol=1e-12)
    # lse of one shard over everything: log2 Σ exp(s) by brute force for one (row, head)
    o1, l1 = OL.paged_decode_attention_lse(q, kc, vc, bt, sl, Hq, Hkv, D)
    b, h = 0, 3
    kv = h // (Hq // Hkv)
    s_t = [float(kc[bt[b][t // 16], kv, t % 16] @ q[b, h * D:(h + 1) * D]) / np.sqrt(D) for t in range(sl[b])]
    assert abs(l1[b, h] - np.log2(np.sum(np.exp(s_t)))) < 1e-12
