"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no norm, no GEMM, no RoPE, no
softmax, no DAG/placement logic). It only draws random numbers, encodes them
as bf16 bit patterns and lays out paged-KV bookkeeping (block tables), so that
`oracle/` and the CUDA path can consume byte-identical inputs without sharing
code (task rule ③; recipe in DESIGN.md §"Input recipe").

Distributions (SURVEY §8(d) "Synthetic inputs"):
  weights N(0, 1/K) (W_o, W_d further x 1/sqrt(2L)); gamma = 1 + 0.1 N(0,1);
  residual x and pre-filled KV N(0,1); block tables = seeded random page
  permutation (fragmented pool); seed = 0x4B440000 + config_index.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Dict, Optional

import numpy as np

SEED_BASE = 0x4B44_0000


# --------------------------------------------------------------------------
# configurations (shapes only; BASELINE.json "configs", SURVEY §8 notation)
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class DecoderConfig:
    name: str
    hidden: int            # H
    n_heads: int           # Hq
    n_kv_heads: int        # Hkv
    head_dim: int          # D
    ffn: int               # F
    n_layers: int          # L
    batch: int             # B (sequences decoded per step)
    context: int           # C keys attended incl. the new token (R15)
    page: int = 16         # P tokens per KV page
    rope_theta: float = 1e4
    eps: float = 1e-5
    n_micro: int = 1       # N micro-batches per step
    act: str = "bf16"      # activation storage dtype ("bf16" | "fp32", R12/R13)
    config_index: int = 0
    # MoE (a11); 0 = dense
    n_experts: int = 0
    top_k: int = 2
    # Mamba-2 hybrid (a12); attn_every = 0 → all layers attention
    attn_every: int = 0
    ssm_heads: int = 128
    ssm_head_dim: int = 64
    d_state: int = 128
    ssm_groups: int = 8
    d_conv: int = 4

    def is_attn_layer(self, l: int) -> bool:
        """R19: attention at layers l ≡ attn_every−1 (mod attn_every), Mamba-2 elsewhere."""
        return self.attn_every == 0 or l % self.attn_every == self.attn_every - 1

    @property
    def d_inner(self) -> int:
        return self.ssm_heads * self.ssm_head_dim

    @property
    def conv_channels(self) -> int:
        return self.d_inner + 2 * self.ssm_groups * self.d_state

    @property
    def in_proj_dim(self) -> int:
        return 2 * self.d_inner + 2 * self.ssm_groups * self.d_state + self.ssm_heads

    @property
    def group(self) -> int:
        return self.n_heads // self.n_kv_heads

    @property
    def qkv_dim(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    @property
    def m(self) -> int:
        assert self.batch % self.n_micro == 0
        return self.batch // self.n_micro

    @property
    def pages_per_seq(self) -> int:
        return (self.context + self.page - 1) // self.page

    @property
    def seed(self) -> int:
        return SEED_BASE + self.config_index

    def with_(self, **kw) -> "DecoderConfig":
        return replace(self, **kw)


TINY = DecoderConfig("tiny", hidden=256, n_heads=4, n_kv_heads=4, head_dim=64,
                     ffn=1024, n_layers=2, batch=4, context=128,
                     rope_theta=1e4, n_micro=4, config_index=0)
LLAMA8B = DecoderConfig("llama3-8b", hidden=4096, n_heads=32, n_kv_heads=8,
                        head_dim=128, ffn=14336, n_layers=32, batch=64,
                        context=4096, rope_theta=5e5, n_micro=1, config_index=1)
LLAMA70B = DecoderConfig("llama3-70b", hidden=8192, n_heads=64, n_kv_heads=8,
                         head_dim=128, ffn=28672, n_layers=80, batch=128,
                         context=8192, rope_theta=5e5, n_micro=2, config_index=2)
MIXTRAL = DecoderConfig("mixtral-8x7b", hidden=4096, n_heads=32, n_kv_heads=8,
                        head_dim=128, ffn=14336, n_layers=32, batch=128,
                        context=4096, rope_theta=1e6, n_micro=1, config_index=3,
                        n_experts=8, top_k=2)

HYBRID = DecoderConfig("hybrid-mamba2", hidden=4096, n_heads=32, n_kv_heads=8, head_dim=128, ffn=14336,
                       n_layers=32, batch=64, context=4096, rope_theta=5e5, n_micro=1, config_index=4,
                       attn_every=8, ssm_heads=128, ssm_head_dim=64, d_state=128, ssm_groups=8, d_conv=4)
TINY_HYBRID = DecoderConfig("tiny-hybrid", hidden=256, n_heads=4, n_kv_heads=2, head_dim=64, ffn=512,
                            n_layers=4, batch=4, context=64, rope_theta=1e4, n_micro=2, config_index=5,
                            attn_every=2, ssm_heads=8, ssm_head_dim=32, d_state=32, ssm_groups=2, d_conv=4)

CONFIGS = {c.name: c for c in (TINY, LLAMA8B, LLAMA70B, MIXTRAL, HYBRID, TINY_HYBRID)}


# --------------------------------------------------------------------------
# bf16 encoding of drawn numbers (input encoding only)
# --------------------------------------------------------------------------
def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Encode float32 draws as bf16 bit patterns (round-to-nearest-even)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    """Decode bf16 bit patterns (exact)."""
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def normal_bf16(g: np.random.Generator, shape, std: float = 1.0) -> np.ndarray:
    return f32_to_bf16_bits((g.standard_normal(shape, dtype=np.float32) * np.float32(std)))


def normal_f32(g: np.random.Generator, shape, std: float = 1.0) -> np.ndarray:
    return (g.standard_normal(shape, dtype=np.float32) * np.float32(std)).astype(np.float32)


def block_table(g: np.random.Generator, n_seq: int, pages_per_seq: int, n_micro: int = 1) -> np.ndarray:
    """Fragmented page pool: the pool is the concatenation of
    one sub-pool per micro-batch (micro-batch i = sequences [i·m, (i+1)·m));
    inside sub-pool i the page ids are a seeded random permutation, sequence b
    owns perm_i[(b − i·m)·pps : (b − i·m + 1)·pps] + i·m·pps. Ids are global."""
    assert n_seq % n_micro == 0
    m = n_seq // n_micro
    sub = m * pages_per_seq
    out = np.empty((n_seq, pages_per_seq), dtype=np.int32)
    for i in range(n_micro):
        perm = g.permutation(sub).astype(np.int32) + i * sub
        out[i * m:(i + 1) * m] = perm.reshape(m, pages_per_seq)
    return out


# --------------------------------------------------------------------------
# decoder inputs for parity-sized runs (host generated)
# --------------------------------------------------------------------------
@dataclass
class LayerWeights:
    w_qkv: np.ndarray   # bf16 bits [qkv_dim, H], rows kv-group interleaved (R12)
    w_o: np.ndarray     # bf16 bits [H, Hq*D]
    w_gu: np.ndarray    # bf16 bits [2F, H], gate/up 64-row block interleaved (R12)
    w_d: np.ndarray     # bf16 bits [H, F]
    gamma1: np.ndarray  # bf16 bits [H]
    gamma2: np.ndarray  # bf16 bits [H]
    # MoE (only when cfg.n_experts > 0): router fp32, experts bf16
    w_router: Optional[np.ndarray] = None   # f32 [E, H]
    w_gu_e: Optional[np.ndarray] = None     # bf16 bits [E, 2F, H]
    w_d_e: Optional[np.ndarray] = None      # bf16 bits [E, H, F]


@dataclass
class MambaWeights:
    gamma: np.ndarray    # bf16 bits [H]   pre-norm
    w_in: np.ndarray     # bf16 bits [2·d_inner + 2·G·N + nheads, H]  rows [z | xBC | dt]
    conv_w: np.ndarray   # bf16 bits [conv_channels, d_conv]
    conv_b: np.ndarray   # bf16 bits [conv_channels]
    dt_bias: np.ndarray  # f32 [nheads]
    A_log: np.ndarray    # f32 [nheads]
    D: np.ndarray        # f32 [nheads]
    norm_w: np.ndarray   # bf16 bits [d_inner]  gated RMSNorm weight
    w_out: np.ndarray    # bf16 bits [H, d_inner]


def make_mamba_weights(g: np.random.Generator, cfg: DecoderConfig) -> MambaWeights:
    H, di, L = cfg.hidden, cfg.d_inner, cfg.n_layers
    nh = cfg.ssm_heads
    u = g.uniform(1e-3, 0.1, nh)
    return MambaWeights(
        gamma=f32_to_bf16_bits(1.0 + 0.1 * g.standard_normal(H, dtype=np.float32)),
        w_in=normal_bf16(g, (cfg.in_proj_dim, H), 1.0 / math.sqrt(H)),
        conv_w=normal_bf16(g, (cfg.conv_channels, cfg.d_conv), 0.5),
        conv_b=normal_bf16(g, (cfg.conv_channels,), 0.5),
        dt_bias=np.log(np.expm1(u)).astype(np.float32),          # softplus⁻¹(U[1e-3, 0.1])
        A_log=np.log(g.uniform(1.0, 16.0, nh)).astype(np.float32),
        D=np.ones(nh, np.float32),
        norm_w=f32_to_bf16_bits(1.0 + 0.1 * g.standard_normal(di, dtype=np.float32)),
        w_out=normal_bf16(g, (H, di), 1.0 / math.sqrt(2.0 * L) / math.sqrt(di)),
    )


@dataclass
class DecoderInputs:
    cfg: DecoderConfig
    layers: list
    x: np.ndarray             # f32 [B, H] residual stream entering layer 0
    k_cache: list             # per layer bf16 bits [n_pages, Hkv, P, D] (HND, R12)
    v_cache: list
    block_table: np.ndarray   # int32 [B, pages_per_seq]
    seq_len: np.ndarray       # int32 [B] (= C, R15)
    conv_state: Optional[list] = None  # per layer (Mamba layers) bf16 bits [B, conv_channels, d_conv-1]
    ssm_state: Optional[list] = None   # per layer (Mamba layers) f32 [B, nheads, head_dim, d_state]


def make_layer_weights(g: np.random.Generator, cfg: DecoderConfig) -> LayerWeights:
    H, F, L = cfg.hidden, cfg.ffn, cfg.n_layers
    HqD = cfg.n_heads * cfg.head_dim
    out_scale = 1.0 / math.sqrt(2.0 * L)
    lw = LayerWeights(
        w_qkv=normal_bf16(g, (cfg.qkv_dim, H), 1.0 / math.sqrt(H)),
        w_o=normal_bf16(g, (H, HqD), out_scale / math.sqrt(HqD)),
        w_gu=normal_bf16(g, (2 * F, H), 1.0 / math.sqrt(H)),
        w_d=normal_bf16(g, (H, F), out_scale / math.sqrt(F)),
        gamma1=f32_to_bf16_bits(1.0 + 0.1 * g.standard_normal(H, dtype=np.float32)),
        gamma2=f32_to_bf16_bits(1.0 + 0.1 * g.standard_normal(H, dtype=np.float32)),
    )
    if cfg.n_experts:
        E = cfg.n_experts
        lw.w_router = normal_f32(g, (E, H), 1.0 / math.sqrt(H))
        lw.w_gu_e = normal_bf16(g, (E, 2 * F, H), 1.0 / math.sqrt(H))
        lw.w_d_e = normal_bf16(g, (E, H, F), out_scale / math.sqrt(F))
        lw.w_gu = None
        lw.w_d = None
    return lw


def make_decoder_inputs(cfg: DecoderConfig, seed: Optional[int] = None) -> DecoderInputs:
    g = rng(cfg.seed if seed is None else seed)
    layers = [make_layer_weights(g, cfg) if cfg.is_attn_layer(l) else make_mamba_weights(g, cfg)
              for l in range(cfg.n_layers)]
    x = normal_f32(g, (cfg.batch, cfg.hidden))
    pps = cfg.pages_per_seq
    bt = block_table(g, cfg.batch, pps, cfg.n_micro)
    n_pages = cfg.batch * pps
    kshape = (n_pages, cfg.n_kv_heads, cfg.page, cfg.head_dim)
    kc = [normal_bf16(g, kshape) if cfg.is_attn_layer(l) else None for l in range(cfg.n_layers)]
    vc = [normal_bf16(g, kshape) if cfg.is_attn_layer(l) else None for l in range(cfg.n_layers)]
    seq_len = np.full(cfg.batch, cfg.context, dtype=np.int32)
    conv = ssm = None
    if cfg.attn_every:
        conv = [None if cfg.is_attn_layer(l) else normal_bf16(g, (cfg.batch, cfg.conv_channels, cfg.d_conv - 1))
                for l in range(cfg.n_layers)]
        ssm = [None if cfg.is_attn_layer(l) else
               normal_f32(g, (cfg.batch, cfg.ssm_heads, cfg.ssm_head_dim, cfg.d_state), 0.1)
               for l in range(cfg.n_layers)]
    return DecoderInputs(cfg, layers, x, kc, vc, bt, seq_len, conv, ssm)


# --------------------------------------------------------------------------
# on-device bulk generation for throughput runs (46 GB of 8B-shaped state);
# values never feed a stored expected value — parity at full size samples
# these tensors back to the host and recomputes with the oracle.
# --------------------------------------------------------------------------
def device_normal_(t, seed: int, std: float = 1.0):
    """Fill a torch tensor (any float dtype, any device) with N(0, std^2)."""
    import torch
    gen = torch.Generator(device=t.device)
    gen.manual_seed(int(seed) & 0x7FFFFFFFFFFFFFFF)
    if t.dtype in (torch.float32, torch.float64):
        t.normal_(0.0, std, generator=gen)
    else:
        tmp = torch.empty(t.shape, dtype=torch.float32, device=t.device)
        # chunk to bound the fp32 staging footprint
        flat_t = t.view(-1)
        flat = tmp.view(-1)
        flat.normal_(0.0, std, generator=gen)
        flat_t.copy_(flat)
    return t
