"""Oracle — prefill-phase decoder math in fp64 (test infrastructure only; see
oracle/__init__.py). SURVEY §8(f) f4: the prefill kernel graph on the same
DAG/placement machinery (§2: prefill kernels include the
memory-bound cublasGemv and the compute-bound FlashAttention).

A prefill step processes S prompt tokens of each of B sequences at once: the
same Llama-style layer as decode (C1.1-C1.11) with every token a row of the
GEMMs, RoPE at each token's own position t in [0, S), the rotated keys and
the values written to the paged cache at slots 0..S-1, and CAUSAL
self-attention (token t attends keys 0..t of its own sequence). Storage
precision follows reading R12 exactly as in layer.py: every kernel output is
rounded to the activation dtype, the residual stream is fp32.

Token row r of every activation is (sequence b, position t) with r = b*S + t.
"""
from __future__ import annotations

import math

import numpy as np

from .layer import (add_rmsnorm, bf16_to_f64, linear, residual_add, rope_neox, silu_mul_blocked,
                    split_qkv_grouped, store)


def rope_prefill(qkv, S, block_table, k_cache, v_cache, n_heads, n_kv, D, theta, page=16, act="bf16"):
    """RoPE at every prompt position and the paged-cache fill (a5 for a
    prompt, C1.3-C1.4): row r = b*S + t gets q, k rotated by t·θ^(-2i/D);
    (k_rot, v) are written to slot t of sequence b (page block_table[b][t//P],
    offset t mod P). Caches [n_pages, Hkv, P, D] are modified in place (values
    stored in `act`). Returns q_rot [B*S, Hq*D] stored in `act`."""
    rows = qkv.shape[0]
    q_out = np.zeros((rows, n_heads * D))
    for r in range(rows):
        b, t = divmod(r, S)
        q, k, v = split_qkv_grouped(qkv[r], n_heads, n_kv, D)
        for h in range(n_heads):
            q_out[r, h * D:(h + 1) * D] = rope_neox(q[h], t, theta)
        pg, off = int(block_table[b][t // page]), t % page
        for g in range(n_kv):
            k_cache[pg, g, off, :] = store(rope_neox(k[g], t, theta), act)
            v_cache[pg, g, off, :] = store(v[g], act)
    return store(q_out, act)


def prefill_attention(q, k_cache, v_cache, block_table, S, n_heads, n_kv, D, page=16, act="bf16"):
    """Causal GQA self-attention over the prompt (FlashAttention's function,
    P:190): for row r = b*S + t and q-head h (kv head g = ⌊h/(Hq/Hkv)⌋),
    s_j = q·k_j/√D for keys j ≤ t of sequence b (read from the paged cache);
    p = softmax(s) (max-subtracted); out = Σ_j p_j v_j.
    q [B*S, Hq*D]; returns [B*S, Hq*D] stored in `act`."""
    rows = q.shape[0]
    B = rows // S
    G = n_heads // n_kv
    out = np.zeros((rows, n_heads * D))
    scale = 1.0 / math.sqrt(D)
    for b in range(B):
        pages = [int(block_table[b][j // page]) for j in range(S)]
        offs = [j % page for j in range(S)]
        for g in range(n_kv):
            K = np.asarray(k_cache[pages, g, offs, :], np.float64)   # [S, D]
            V = np.asarray(v_cache[pages, g, offs, :], np.float64)
            for j in range(G):
                h = g * G + j
                Q = np.asarray(q[b * S:(b + 1) * S, h * D:(h + 1) * D], np.float64)  # [S, D]
                s = (Q @ K.T) * scale                                      # [S, S]
                s = np.where(np.tril(np.ones((S, S), dtype=bool)), s, -np.inf)
                p = np.exp(s - s.max(axis=1, keepdims=True))
                p /= p.sum(axis=1, keepdims=True)
                out[b * S:(b + 1) * S, h * D:(h + 1) * D] = p @ V
    return store(out, act)


def prefill_layer(r, delta_prev, lw, k_cache, v_cache, block_table, S, cfg, act="bf16"):
    """One decoder layer over the prompt tokens in program order (the prefill
    graph's kernels: norm1, QKV, RoPE+cache fill, causal attention, O, norm2,
    gate_up, SiLU·mul, down). Returns (r, d) as layer.decoder_layer."""
    H, Hq, Hkv, D = cfg.hidden, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    dec = bf16_to_f64
    r, h1 = add_rmsnorm(r, delta_prev, dec(lw.gamma1), cfg.eps, act)
    qkv = linear(h1, dec(lw.w_qkv), act)
    q = rope_prefill(qkv, S, block_table, k_cache, v_cache, Hq, Hkv, D, cfg.rope_theta, cfg.page, act)
    attn = prefill_attention(q, k_cache, v_cache, block_table, S, Hq, Hkv, D, cfg.page, act)
    o = linear(attn, dec(lw.w_o), act)
    r, h2 = add_rmsnorm(r, o, dec(lw.gamma2), cfg.eps, act)
    gu = linear(h2, dec(lw.w_gu), act)
    a = silu_mul_blocked(gu, act=act)
    d = linear(a, dec(lw.w_d), act)
    return r, d


def prefill_step(inp, S, act="bf16", layers=None):
    """Prefill of S prompt tokens for each of the B sequences of `inp`
    (synth.DecoderInputs; its residual x must have B*S rows, row b*S + t the
    embedding of token t of sequence b). Caches are decoded from bf16, filled
    at slots 0..S-1 on copies and returned. Returns (r_out [B*S, H], kcs, vcs)."""
    cfg = inp.cfg
    L = cfg.n_layers if layers is None else layers
    r = np.asarray(inp.x, np.float64)
    assert r.shape[0] % S == 0
    d = None
    kcs, vcs = [], []
    for l in range(L):
        kc = store(bf16_to_f64(inp.k_cache[l]), act)
        vc = store(bf16_to_f64(inp.v_cache[l]), act)
        r, d = prefill_layer(r, d, inp.layers[l], kc, vc, inp.block_table, S, cfg, act)
        kcs.append(kc)
        vcs.append(vc)
    return residual_add(r, d), kcs, vcs
