"""Pins of the prefill oracle (oracle/prefill.py) against
things other than itself:
  * the pinned DECODE oracle: prefill of S tokens ends, for its last token,
    exactly where prefill of S-1 tokens followed by one decode step (C1,
    decoder_step, a different code path: single-query attention, RoPE at
    seq_len-1) ends — and leaves the same cache slots;
  * causality: no output of a token depends on later tokens (bitwise);
  * closed forms of causal attention (token 0 → v_0; identical keys → the
    running mean of V)."""
import math

import numpy as np
import pytest

import synth
from oracle import layer as OL, prefill as PF

CFG = synth.DecoderConfig("tiny-prefill", hidden=64, n_heads=4, n_kv_heads=2, head_dim=16, ffn=128,
                          n_layers=2, batch=2, context=12, page=4, rope_theta=1e4, n_micro=1, config_index=7)


def prompt_inputs(cfg, S, seed=11):
    inp = synth.make_decoder_inputs(cfg, seed=seed)
    g = np.random.default_rng(seed + 1)
    inp.x = g.standard_normal((cfg.batch * S, cfg.hidden)).astype(np.float32)
    return inp


def to_bits(vals):
    return synth.f32_to_bf16_bits(np.asarray(vals, np.float32))


@pytest.mark.parametrize("S", [1, 5, 8])
def test_prefill_last_token_equals_prefill_then_decode(S):
    """P(S)[last] == decode(P(S-1) caches, token S-1): the prefill graph and the
    decode graph compute the same function of the prompt (causal attention
    over slots 0..t is exactly decode attention at seq_len t+1)."""
    cfg = CFG
    inp = prompt_inputs(cfg, S)
    r_full, kc_full, vc_full = PF.prefill_step(inp, S)
    # prefill of the first S-1 tokens, then one decode step on token S-1
    B, H = cfg.batch, cfg.hidden
    x_tok = inp.x.reshape(B, S, H)
    if S > 1:
        inp_p = prompt_inputs(cfg, S - 1)
        inp_p.x = np.ascontiguousarray(x_tok[:, :S - 1]).reshape(B * (S - 1), H)
        _, kc_p, vc_p = PF.prefill_step(inp_p, S - 1)
        kbits = [to_bits(k) for k in kc_p]
        vbits = [to_bits(v) for v in vc_p]
    else:
        kbits, vbits = inp.k_cache, inp.v_cache
    dec = synth.DecoderInputs(cfg, inp.layers, np.ascontiguousarray(x_tok[:, S - 1]), kbits, vbits,
                              inp.block_table, np.full(B, S, np.int32))
    r_dec, kc_dec, vc_dec = OL.decoder_step(dec)
    np.testing.assert_allclose(r_full.reshape(B, S, H)[:, S - 1], r_dec, rtol=0, atol=1e-9)
    # and the cache slots 0..S-1 agree
    for l in range(cfg.n_layers):
        for b in range(B):
            for t in range(S):
                pg, off = int(inp.block_table[b][t // cfg.page]), t % cfg.page
                np.testing.assert_allclose(kc_full[l][pg, :, off], kc_dec[l][pg, :, off], rtol=0, atol=1e-9)
                np.testing.assert_allclose(vc_full[l][pg, :, off], vc_dec[l][pg, :, off], rtol=0, atol=1e-9)


def test_causality_later_tokens_do_not_change_earlier_outputs():
    cfg, S, t0 = CFG, 7, 3
    inp = prompt_inputs(cfg, S)
    r1, _, _ = PF.prefill_step(inp, S)
    x = inp.x.reshape(cfg.batch, S, cfg.hidden).copy()
    x[:, t0 + 1:] += 5.0
    inp.x = x.reshape(cfg.batch * S, cfg.hidden)
    r2, _, _ = PF.prefill_step(inp, S)
    a = r1.reshape(cfg.batch, S, -1)
    b = r2.reshape(cfg.batch, S, -1)
    assert np.array_equal(a[:, :t0 + 1], b[:, :t0 + 1])
    assert not np.allclose(a[:, t0 + 1:], b[:, t0 + 1:])


def test_causal_attention_closed_forms():
    """Token 0 attends only itself (out = v_0); with identical keys every token
    t gets the running mean of v_0..v_t (uniform softmax over the window)."""
    B, S, Hq, Hkv, D, P = 2, 6, 4, 2, 8, 4
    pps = (S + P - 1) // P
    bt = np.arange(B * pps, dtype=np.int32).reshape(B, pps)[:, ::-1].copy()  # pages in reverse order
    g = np.random.default_rng(3)
    kc = np.zeros((B * pps, Hkv, P, D))
    vc = np.zeros((B * pps, Hkv, P, D))
    V = g.standard_normal((B, S, Hkv, D))
    kconst = g.standard_normal((Hkv, D))
    for b in range(B):
        for t in range(S):
            kc[bt[b][t // P], :, t % P] = kconst
            vc[bt[b][t // P], :, t % P] = V[b, t]
    q = g.standard_normal((B * S, Hq * D))
    out = PF.prefill_attention(q, kc, vc, bt, S, Hq, Hkv, D, P, act="f64")
    G = Hq // Hkv
    for b in range(B):
        for t in range(S):
            for h in range(Hq):
                want = V[b, : t + 1, h // G].mean(axis=0)
                np.testing.assert_allclose(out[b * S + t, h * D:(h + 1) * D], want, rtol=1e-12, atol=1e-12)
    # distinct keys: token 0 → v_0 exactly
    kc2 = g.standard_normal(kc.shape)
    out2 = PF.prefill_attention(q, kc2, vc, bt, S, Hq, Hkv, D, P, act="f64")
    for b in range(B):
        for h in range(Hq):
            np.testing.assert_allclose(out2[b * S, h * D:(h + 1) * D], V[b, 0, h // G], rtol=1e-12, atol=1e-12)


def test_rope_prefill_positions_and_slots():
    """q of token t is rotated by t radians·θ^(-2i/D) (D=2: a plain rotation by
    t rad, i=0), and (k_rot, v) land in slot t of the sequence's pages."""
    Hq = Hkv = 1
    D, P, S, B = 2, 4, 6, 1
    pps = 2
    bt = np.array([[1, 0]], dtype=np.int32)
    qkv = np.zeros((S, 3 * D))
    for t in range(S):
        qkv[t] = [1.0, 0.0, 0.0, 1.0, 2.0 + t, -t]   # q = (1, 0), k = (0, 1), v
    kc = np.zeros((B * pps, Hkv, P, D))
    vc = np.zeros((B * pps, Hkv, P, D))
    q = PF.rope_prefill(qkv, S, bt, kc, vc, Hq, Hkv, D, theta=1e4, page=P, act="f64")
    for t in range(S):
        np.testing.assert_allclose(q[t], [math.cos(t), math.sin(t)], rtol=0, atol=1e-15)
        pg, off = bt[0][t // P], t % P
        np.testing.assert_allclose(kc[pg, 0, off], [-math.sin(t), math.cos(t)], rtol=0, atol=1e-15)
        np.testing.assert_allclose(vc[pg, 0, off], [2.0 + t, -t], rtol=0, atol=0)
