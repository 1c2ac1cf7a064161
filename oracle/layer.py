"""Oracle — decoder-layer math in fp64 (test infrastructure only; see oracle/__init__.py).

The paper fixes no model math (it runs vLLM's kernels); the decoder
layer here is the standard Llama-style decode layer the paper's workloads use
(Llama-3 8B P:490). Arithmetic is fp64. Storage precision
follows reading R12: every kernel output is rounded to the activation dtype
(bf16 or fp32) except the residual stream, which is stored in fp32.

All functions take plain numpy arrays. bf16 inputs arrive as uint16 bit
patterns and are decoded with `bf16_to_f64`.
"""
from __future__ import annotations

import math

import numpy as np


# ---------------------------------------------------------------- storage
def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    """Exact decode of bf16 bit patterns."""
    u = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    return u.view(np.float32).astype(np.float64)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round to the nearest bf16 value (ties to even), via fp32 (R12)."""
    f = np.asarray(x, dtype=np.float64).astype(np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def round_f32(x: np.ndarray) -> np.ndarray:
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def store(x: np.ndarray, act: str) -> np.ndarray:
    """Round a kernel output to its storage dtype (R12/R13)."""
    if act == "bf16":
        return round_bf16(x)
    if act == "fp32":
        return round_f32(x)
    if act == "f64":
        return np.asarray(x, dtype=np.float64)
    raise ValueError(act)


# ---------------------------------------------------------------- a3
def add_rmsnorm(r, delta, gamma, eps, act="bf16"):
    """Fused residual add + RMSNorm (C1.1).

    r' = r + delta   (stored fp32: the residual stream, R12)
    h  = r' / sqrt(mean_j r'_j^2 + eps) * gamma   (stored in `act`)
    `delta=None` means no add (first layer). Returns (r', h).
    """
    r = np.asarray(r, dtype=np.float64)
    rn = r if delta is None else r + np.asarray(delta, dtype=np.float64)
    rn = round_f32(rn)
    ms = np.mean(rn * rn, axis=-1, keepdims=True)
    h = rn / np.sqrt(ms + eps) * np.asarray(gamma, dtype=np.float64)
    return rn, store(h, act)


def residual_add(r, delta):
    """Final residual add after the last layer (C1.11); fp32 storage."""
    return round_f32(np.asarray(r, np.float64) + np.asarray(delta, np.float64))


# ---------------------------------------------------------------- a4/a7/a9/a10
def linear(x, w, act="bf16"):
    """y = x · Wᵀ with W row-major [N_out, K] (nn.Linear convention, C1.2)."""
    y = np.asarray(x, np.float64) @ np.asarray(w, np.float64).T
    return store(y, act)


# ---------------------------------------------------------------- a5
def rope_freqs(pos: int, head_dim: int, theta: float):
    """cos/sin of pos·theta^(−2i/D), i < D/2, in fp64 (R12)."""
    i = np.arange(head_dim // 2, dtype=np.float64)
    ang = float(pos) * np.power(float(theta), -2.0 * i / head_dim)
    return np.cos(ang), np.sin(ang)


def rope_neox(x, pos: int, theta: float):
    """NeoX / rotate-half RoPE on one head vector x[D] (C1.3):
    x'_i = x_i c_i − x_{i+D/2} s_i ;  x'_{i+D/2} = x_{i+D/2} c_i + x_i s_i."""
    x = np.asarray(x, np.float64)
    D = x.shape[-1]
    c, s = rope_freqs(pos, D, theta)
    a, b = x[..., : D // 2], x[..., D // 2:]
    return np.concatenate([a * c - b * s, b * c + a * s], axis=-1)


def split_qkv_grouped(qkv_row, n_heads, n_kv, D):
    """Split one token's qkv row in the kv-group-interleaved layout (R12):
    for g < Hkv: [q_{gG}, …, q_{gG+G−1}, k_g, v_g], each D wide.
    Returns q [Hq, D], k [Hkv, D], v [Hkv, D]."""
    G = n_heads // n_kv
    blk = np.asarray(qkv_row).reshape(n_kv, G + 2, D)
    q = blk[:, :G, :].reshape(n_heads, D)
    return q, blk[:, G, :], blk[:, G + 1, :]


def rope_append(qkv, pos, block_table, k_cache, v_cache, n_heads, n_kv, D,
                theta, page=16, act="bf16"):
    """RoPE on q and k, then append (k_rot, v) to the paged cache at `pos`
    (C1.3–C1.4). qkv [m, qkv_dim]; pos [m] int; block_table
    [m, pages]; caches [n_pages, Hkv, P, D] (HND, R12) modified in place
    (values stored in `act`). Returns q_rot [m, Hq*D] stored in `act`."""
    m = qkv.shape[0]
    q_out = np.zeros((m, n_heads * D))
    for b in range(m):
        q, k, v = split_qkv_grouped(qkv[b], n_heads, n_kv, D)
        p = int(pos[b])
        for h in range(n_heads):
            q_out[b, h * D:(h + 1) * D] = rope_neox(q[h], p, theta)
        pg = int(block_table[b][p // page])
        off = p % page
        for g in range(n_kv):
            k_cache[pg, g, off, :] = store(rope_neox(k[g], p, theta), act)
            v_cache[pg, g, off, :] = store(v[g], act)
    return store(q_out, act)


# ---------------------------------------------------------------- a6
def paged_decode_attention(q, k_cache, v_cache, block_table, seq_len,
                           n_heads, n_kv, D, page=16, act="bf16"):
    """Single-query decode attention over a paged cache (C1.5):
    for sequence b and q-head h with kv head g = ⌊h / (Hq/Hkv)⌋,
    s_t = q·k_t / √D for t < seq_len[b]; p = softmax(s) (max-subtracted);
    out = Σ_t p_t v_t. No mask beyond the length, no sliding window.
    q [m, Hq*D]; returns [m, Hq*D] stored in `act`."""
    m = q.shape[0]
    G = n_heads // n_kv
    out = np.zeros((m, n_heads * D))
    scale = 1.0 / math.sqrt(D)
    for b in range(m):
        C = int(seq_len[b])
        pages = [int(block_table[b][t // page]) for t in range(C)]
        offs = [t % page for t in range(C)]
        for g in range(n_kv):
            K = np.asarray(k_cache[pages, g, offs, :], np.float64)   # [C, D]
            V = np.asarray(v_cache[pages, g, offs, :], np.float64)
            for j in range(G):
                h = g * G + j
                qh = np.asarray(q[b, h * D:(h + 1) * D], np.float64)
                s = (K @ qh) * scale
                p = np.exp(s - s.max())
                p /= p.sum()
                out[b, h * D:(h + 1) * D] = p @ V
    return store(out, act)


def paged_decode_attention_lse(q, k_cache, v_cache, block_table, seq_len, n_heads, n_kv, D, page=16):
    """C1.5 plus the base-2 log-sum-exp of the scaled scores per (row, head):
    lse2 = log2 Σ_t exp(s_t), s_t = q·k_t/√D (−inf for an empty context, whose
    output is 0). Exact fp64; the KV-shard partial of f2."""
    m = q.shape[0]
    G = n_heads // n_kv
    out = np.zeros((m, n_heads * D))
    lse = np.full((m, n_heads), -np.inf)
    scale = 1.0 / math.sqrt(D)
    for b in range(m):
        C = int(seq_len[b])
        if C == 0:
            continue
        pages = [int(block_table[b][t // page]) for t in range(C)]
        offs = [t % page for t in range(C)]
        for g in range(n_kv):
            K = np.asarray(k_cache[pages, g, offs, :], np.float64)
            V = np.asarray(v_cache[pages, g, offs, :], np.float64)
            for j in range(G):
                h = g * G + j
                s = (K @ np.asarray(q[b, h * D:(h + 1) * D], np.float64)) * scale
                mx = s.max()
                e = np.exp(s - mx)
                out[b, h * D:(h + 1) * D] = (e / e.sum()) @ V
                lse[b, h] = (mx + math.log(e.sum())) / math.log(2.0)
    return out, lse


def lse_merge(outs, lses, D):
    """Merge attention partials over disjoint key sets (f2): with weights
    w_s = 2^(lse_s − max_s lse_s), out = Σ_s w_s·out_s / Σ_s w_s — the softmax
    over the union of the key sets written out (shards in index order)."""
    lses = np.asarray(lses, np.float64)           # [S, m, H]
    outs = np.asarray(outs, np.float64)           # [S, m, H*D]
    S, m, H = lses.shape
    M = lses.max(axis=0)
    w = np.where(np.isfinite(lses), np.exp2(lses - np.where(np.isfinite(M), M, 0.0)), 0.0)
    num = (w[:, :, :, None] * outs.reshape(S, m, H, D)).sum(axis=0)
    den = w.sum(axis=0)[:, :, None]
    return np.where(den > 0, num / np.where(den > 0, den, 1.0), 0.0).reshape(m, H * D)


# ---------------------------------------------------------------- a8
def silu(x):
    x = np.asarray(x, np.float64)
    return x / (1.0 + np.exp(-x))


def silu_mul_blocked(gu, block=64, act="bf16"):
    """a = silu(g) · u with gate/up 64-column block interleave (C1.9, R12):
    gu[:, 2jB : 2jB+B] is gate block j, gu[:, 2jB+B : 2jB+2B] is up block j,
    a[:, jB : jB+B] = silu(gate_j) · up_j."""
    gu = np.asarray(gu, np.float64)
    m, two_f = gu.shape
    F = two_f // 2
    a = np.zeros((m, F))
    for j in range(F // block):
        g = gu[:, 2 * j * block: 2 * j * block + block]
        u = gu[:, 2 * j * block + block: 2 * j * block + 2 * block]
        a[:, j * block:(j + 1) * block] = silu(g) * u
    return store(a, act)


# ---------------------------------------------------------------- a11 (MoE)
def moe_route(h, w_router, top_k=2):
    """Router + top-k (C1.12): logits = h·W_rᵀ (fp32 router, computed here in
    fp64), top-k by logit (ties → lower expert index), weights = softmax over
    the k selected logits. Returns (idx [m,k] ascending by rank, w [m,k])."""
    logits = np.asarray(h, np.float64) @ np.asarray(w_router, np.float64).T
    m, E = logits.shape
    idx = np.zeros((m, top_k), dtype=np.int64)
    wts = np.zeros((m, top_k))
    for b in range(m):
        order = sorted(range(E), key=lambda e: (-logits[b, e], e))[:top_k]
        sel = logits[b, order]
        p = np.exp(sel - sel.max())
        idx[b] = order
        wts[b] = p / p.sum()
    return idx, wts


def moe_ffn(h, idx, wts, w_gu_e, w_d_e, act="bf16"):
    """Per-expert SwiGLU and weighted combine (C1.12): for each row b,
    out_b = Σ over its selected experts e in ASCENDING expert order of
    w_{b,e} · (silu·mul(h_b W_gu,eᵀ)) W_d,eᵀ. Expert outputs are stored in
    `act` (they are kernel outputs) before the fp64 weighted sum."""
    h = np.asarray(h, np.float64)
    m = h.shape[0]
    H = w_d_e.shape[1]
    out = np.zeros((m, H))
    for b in range(m):
        pairs = sorted(zip(idx[b].tolist(), wts[b].tolist()))
        for e, w in pairs:
            gu = linear(h[b:b + 1], w_gu_e[e], act)
            a = silu_mul_blocked(gu, act=act)
            y = linear(a, w_d_e[e], act)
            out[b] += w * y[0]
    return store(out, act)


# ---------------------------------------------------------------- a12 (SSM)
def softplus(x):
    x = np.asarray(x, np.float64)
    return np.where(x > 20.0, x, np.log1p(np.exp(np.minimum(x, 20.0))))


def mamba_conv_step(xbc, conv_state, conv_w, conv_b, act="bf16"):
    """Causal depthwise conv1d, one decode step (C1.13, SURVEY a12 "conv: shift
    state, 4-tap dot, SiLU"). xbc [m, Ch] new inputs; conv_state [m, Ch, W-1]
    previous inputs oldest first; conv_w [Ch, W]; conv_b [Ch].
    window = [state, x]; out = silu(Σ_w window_w · conv_w[:, w] + b);
    new_state = window[1:]. Returns (out stored in act, new_state stored in act)."""
    win = np.concatenate([np.asarray(conv_state, np.float64), np.asarray(xbc, np.float64)[:, :, None]], axis=2)
    pre = np.einsum("mcw,cw->mc", win, np.asarray(conv_w, np.float64)) + np.asarray(conv_b, np.float64)
    return store(silu(pre), act), store(win[:, :, 1:], act)


def mamba_ssm_step(x, Bm, Cm, dt, dt_bias, A_log, D, state, nheads, headdim, dstate, ngroups, act="bf16"):
    """Mamba-2 selective-state update, one decode step (C1.13):
    for sequence b, head h, group g(h) = ⌊h / (nheads/ngroups)⌋:
      dt_h = softplus(dt[b,h] + dt_bias[h]);  A_h = −exp(A_log[h]);  dA = exp(dt_h·A_h)
      S ← S·dA + dt_h · x[b,h,:] ⊗ B[b,g,:]        (S: [headdim, dstate], fp32 storage)
      y[b,h,:] = S · C[b,g,:] + D[h] · x[b,h,:]
    x [m, nheads·headdim]; Bm, Cm [m, ngroups·dstate]; dt [m, nheads];
    state [m, nheads, headdim, dstate]. Returns (y stored in act, new state fp32)."""
    m = x.shape[0]
    hpg = nheads // ngroups
    X = np.asarray(x, np.float64).reshape(m, nheads, headdim)
    Bv = np.asarray(Bm, np.float64).reshape(m, ngroups, dstate)
    Cv = np.asarray(Cm, np.float64).reshape(m, ngroups, dstate)
    S = np.asarray(state, np.float64).copy()
    y = np.zeros((m, nheads, headdim))
    for b in range(m):
        for h in range(nheads):
            g = h // hpg
            dth = softplus(dt[b, h] + dt_bias[h])
            dA = np.exp(dth * -np.exp(A_log[h]))
            S[b, h] = S[b, h] * dA + dth * np.outer(X[b, h], Bv[b, g])
            y[b, h] = S[b, h] @ Cv[b, g] + D[h] * X[b, h]
    return store(y.reshape(m, nheads * headdim), act), round_f32(S)


def gated_rmsnorm(y, z, weight, group_size, eps, act="bf16"):
    """Gated RMSNorm of Mamba-2 (C1.13): g = y · silu(z); per group of
    `group_size` channels, out = g / sqrt(mean(g²) + eps) · weight."""
    g = np.asarray(y, np.float64) * silu(z)
    m, n = g.shape
    gg = g.reshape(m, n // group_size, group_size)
    out = gg / np.sqrt(np.mean(gg * gg, axis=-1, keepdims=True) + eps)
    return store(out.reshape(m, n) * np.asarray(weight, np.float64), act)


def mamba_layer(r, delta_prev, mw, conv_state, ssm_state, cfg, act="bf16"):
    """One Mamba-2 decode layer in program order (C1.13): add+RMSNorm →
    in_proj → conv step → SSM step → gated RMSNorm → out_proj. in_proj columns
    are [z (d_inner) | xBC (d_inner + 2·G·N) | dt (nheads)] (Mamba-2 order).
    Returns (r, d, conv_state', ssm_state')."""
    dec = bf16_to_f64
    di, G, N, nh, P = cfg.d_inner, cfg.ssm_groups, cfg.d_state, cfg.ssm_heads, cfg.ssm_head_dim
    r, h = add_rmsnorm(r, delta_prev, dec(mw.gamma), cfg.eps, act)
    zxbcdt = linear(h, dec(mw.w_in), act)
    z = zxbcdt[:, :di]
    xbc = zxbcdt[:, di:2 * di + 2 * G * N]
    dt = zxbcdt[:, 2 * di + 2 * G * N:]
    xc, conv_state = mamba_conv_step(xbc, conv_state, dec(mw.conv_w), dec(mw.conv_b), act)
    y, ssm_state = mamba_ssm_step(xc[:, :di], xc[:, di:di + G * N], xc[:, di + G * N:], dt, mw.dt_bias, mw.A_log,
                                  mw.D, ssm_state, nh, P, N, G, act)
    yn = gated_rmsnorm(y, z, dec(mw.norm_w), di // G, cfg.eps, act)
    d = linear(yn, dec(mw.w_out), act)
    return r, d, conv_state, ssm_state


# ---------------------------------------------------------------- layer
def decoder_layer(r, delta_prev, lw, k_cache, v_cache, block_table, seq_len,
                  cfg, act="bf16"):
    """One decoder layer in program order (C1.1–C1.10). Returns (r, d):
    the residual after the second add and this layer's down-proj output d,
    which folds into the next layer's first add (C1.11)."""
    H, Hq, Hkv, D = cfg.hidden, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    dec = bf16_to_f64
    r, h1 = add_rmsnorm(r, delta_prev, dec(lw.gamma1), cfg.eps, act)
    qkv = linear(h1, dec(lw.w_qkv), act)
    pos = np.asarray(seq_len) - 1
    q = rope_append(qkv, pos, block_table, k_cache, v_cache, Hq, Hkv, D,
                    cfg.rope_theta, cfg.page, act)
    attn = paged_decode_attention(q, k_cache, v_cache, block_table, seq_len,
                                  Hq, Hkv, D, cfg.page, act)
    o = linear(attn, dec(lw.w_o), act)
    r, h2 = add_rmsnorm(r, o, dec(lw.gamma2), cfg.eps, act)
    if cfg.n_experts:
        idx, w = moe_route(h2, lw.w_router, cfg.top_k)
        d = moe_ffn(h2, idx, w, np.stack([dec(x) for x in lw.w_gu_e]),
                    np.stack([dec(x) for x in lw.w_d_e]), act)
    else:
        gu = linear(h2, dec(lw.w_gu), act)
        a = silu_mul_blocked(gu, act=act)
        d = linear(a, dec(lw.w_d), act)
    return r, d


def hybrid_step(inp, act="bf16"):
    """Hybrid decode step: layer l is attention
    (Llama-shaped incl. MLP) when cfg.is_attn_layer(l), else Mamba-2.
    Returns (r_out, conv_states, ssm_states)."""
    cfg = inp.cfg
    r = np.asarray(inp.x, np.float64)
    d = None
    convs, ssms = [], []
    for l in range(cfg.n_layers):
        if cfg.is_attn_layer(l):
            kc = store(bf16_to_f64(inp.k_cache[l]), act)
            vc = store(bf16_to_f64(inp.v_cache[l]), act)
            r, d = decoder_layer(r, d, inp.layers[l], kc, vc, inp.block_table, inp.seq_len, cfg, act)
        else:
            mw = inp.layers[l]
            r, d, cs, ss = mamba_layer(r, d, mw, store(bf16_to_f64(inp.conv_state[l]), act),
                                       round_f32(inp.ssm_state[l]), cfg, act)
            convs.append(cs)
            ssms.append(ss)
    return residual_add(r, d), convs, ssms


def decoder_step(inp, act="bf16", layers=None):
    """Full decode step over `layers` (default all L) for all B sequences,
    micro-batch independent (micro-batching does not change the math).
    Caches are decoded from bf16 (or kept fp32 when act='fp32' — the fp32
    path stores its caches in fp32) and updated in place on copies.
    Returns (r_out [B,H] fp32-valued, caches)."""
    cfg = inp.cfg
    L = cfg.n_layers if layers is None else layers
    r = np.asarray(inp.x, np.float64)
    d = None
    kcs, vcs = [], []
    for l in range(L):
        kc = store(bf16_to_f64(inp.k_cache[l]), act)
        vc = store(bf16_to_f64(inp.v_cache[l]), act)
        r, d = decoder_layer(r, d, inp.layers[l], kc, vc, inp.block_table,
                             inp.seq_len, cfg, act)
        kcs.append(kc)
        vcs.append(vc)
    r = residual_add(r, d)
    return r, kcs, vcs
