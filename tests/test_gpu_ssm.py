"""GPU parity of the Mamba-2 decode kernels and of the
hybrid decoder (attention + Mamba-2 layers) vs the oracle."""
import numpy as np
import pytest

import synth
from oracle import layer as OL
from parity import assert_elementwise

pytestmark = pytest.mark.gpu


def _t():
    import torch
    return torch


def dev_bf16(bits):
    torch = _t()
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def host_f64(t):
    torch = _t()
    if t.dtype == torch.bfloat16:
        return OL.bf16_to_f64(t.view(torch.int16).cpu().numpy().view(np.uint16))
    return t.double().cpu().numpy()


def relerr(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-30))


@pytest.fixture(scope="module")
def kd(cuda_ok):
    from paper_2604_10180_b200 import _kd as K
    return K


SHAPES = [  # rows, nheads, head_dim, d_state, ngroups
    (3, 8, 32, 32, 2),
    (5, 16, 64, 64, 4),
    (64, 128, 64, 128, 8),   # hybrid config, full width
]


@pytest.mark.parametrize("rows,nh,P,N,G", SHAPES)
def test_ssm_kernels_vs_oracle(kd, rows, nh, P, N, G):
    K = kd
    torch = _t()
    W = 4
    cfg = synth.TINY_HYBRID.with_(ssm_heads=nh, ssm_head_dim=P, d_state=N, ssm_groups=G, batch=rows, n_micro=1)
    g = synth.rng(rows * 7 + nh)
    mw = synth.make_mamba_weights(g, cfg)
    di, ch, pin = cfg.d_inner, cfg.conv_channels, cfg.in_proj_dim
    zx = synth.normal_bf16(g, (rows, pin))
    conv_st = synth.normal_bf16(g, (rows, ch, W - 1))
    S0 = synth.normal_f32(g, (rows, nh, P, N), 0.1)
    s = torch.cuda.current_stream().cuda_stream
    a = K.kd_attr_ssm(rows, nh, P, N, G, W, K.KD_BF16, 1e-5)
    zx_d, cw, cb = dev_bf16(zx), dev_bf16(mw.conv_w), dev_bf16(mw.conv_b)
    cst = dev_bf16(conv_st)
    xbc = torch.empty(rows, ch, dtype=torch.bfloat16, device="cuda")
    K.check(K.kd_op_ssm_conv(a, zx_d.data_ptr(), cw.data_ptr(), cb.data_ptr(), cst.data_ptr(), xbc.data_ptr(), s))
    dtb, alog, Dp = (torch.from_numpy(x).cuda() for x in (mw.dt_bias, mw.A_log, mw.D))
    Sd = torch.from_numpy(S0.copy()).cuda()
    y = torch.empty(rows, di, dtype=torch.bfloat16, device="cuda")
    K.check(K.kd_op_ssm_update(a, xbc.data_ptr(), zx_d.data_ptr(), dtb.data_ptr(), alog.data_ptr(), Dp.data_ptr(),
                               Sd.data_ptr(), y.data_ptr(), s))
    nw = dev_bf16(mw.norm_w)
    yn = torch.empty(rows, di, dtype=torch.bfloat16, device="cuda")
    K.check(K.kd_op_gated_norm(a, y.data_ptr(), zx_d.data_ptr(), nw.data_ptr(), yn.data_ptr(), s))
    torch.cuda.synchronize()
    # oracle, step by step on the same inputs
    zxf = OL.bf16_to_f64(zx)
    xc_ref, cst_ref = OL.mamba_conv_step(zxf[:, di:di + ch], OL.bf16_to_f64(conv_st), OL.bf16_to_f64(mw.conv_w),
                                         OL.bf16_to_f64(mw.conv_b), "bf16")
    assert relerr(host_f64(xbc), xc_ref) < 5e-3
    assert_elementwise(host_f64(xbc), xc_ref, 1, 1e-3, "ssm conv xbc")
    assert np.array_equal(host_f64(cst), cst_ref)          # the shift is exact
    y_ref, S_ref = OL.mamba_ssm_step(xc_ref[:, :di], xc_ref[:, di:di + G * N], xc_ref[:, di + G * N:],
                                     zxf[:, di + ch:], mw.dt_bias, mw.A_log, mw.D, S0, nh, P, N, G, "bf16")
    assert relerr(Sd.cpu().numpy(), S_ref) < 5e-3
    assert relerr(host_f64(y), y_ref) < 1e-2
    assert_elementwise(Sd.cpu().numpy(), S_ref, 2, 1e-2, "ssm state")
    assert_elementwise(host_f64(y), y_ref, 2, 2e-2, "ssm y")
    yn_ref = OL.gated_rmsnorm(y_ref, zxf[:, :di], OL.bf16_to_f64(mw.norm_w), di // G, 1e-5, "bf16")
    assert relerr(host_f64(yn), yn_ref) < 1e-2
    assert_elementwise(host_f64(yn), yn_ref, 2, 2e-2, "gated norm")


def test_hybrid_decoder_vs_oracle_and_disaggregated_bitwise(kd):
    from paper_2604_10180_b200 import decoder as DEC
    cfg = synth.TINY_HYBRID
    inp = synth.make_decoder_inputs(cfg)
    dg = DEC.DecoderGraph(cfg)
    mono = DEC.DecoderRuntime(dg, [0] * dg.g.num_kernels, 1, [0], inputs=inp)
    mono.step()
    mono.sync()
    r_ref, _, _ = OL.hybrid_step(inp, act="bf16")
    assert relerr(mono.residual(), r_ref) < 2e-2
    dg2 = DEC.DecoderGraph(cfg)
    dis = DEC.DecoderRuntime(dg2, dg2.role_assign(0, 1), 2, [0, 0], inputs=inp)
    dis.step()
    dis.sync()
    dis.rt.check()
    assert np.array_equal(mono.residual(), dis.residual())
