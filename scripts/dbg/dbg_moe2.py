import sys, os; sys.path.insert(0, "/root/repo")
import synth, numpy as np
from paper_2604_10180_b200 import decoder as DEC
cfg = synth.TINY.with_(n_experts=4, top_k=2, n_micro=2)
inp = synth.make_decoder_inputs(cfg)
dg = DEC.DecoderGraph(cfg)
g = os.environ.get("G", "1") == "1"
rt = DEC.DecoderRuntime(dg, [0]*dg.g.num_kernels, 1, [0], inputs=inp, use_graph=g)
for _ in range(3): rt.step()
rt.sync(); print("ok graph=", g, np.abs(rt.residual()).max())
