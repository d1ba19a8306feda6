"""Run one JIT conv launch sequence (for ncu): layer of config 2, batch N, tile env as set."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1608_01409_b200 import skc  # noqa: E402
import workloads as wl  # noqa: E402
layer, N = sys.argv[1], int(sys.argv[2])
kern = int(sys.argv[3]) if len(sys.argv) > 3 else skc.SKC_KERNEL_JIT
cfg = wl.CONFIGS[2]
li = [L.name for L in cfg.layers].index(layer)
L = cfg.layers[li]
w = wl.gen_weights(2, li, L)
x = torch.from_numpy(wl.gen_input(2, li, L, 0, N)).cuda()
j = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups, kern)
if os.environ.get("SKC_ONE_TUNE", "0") == "1":  # the launch schedule bench.py would use
    print("tuned", j.tune(N), j.plan.info()["jit_sched"])
xp = torch.empty(j.padded_shape(N), device="cuda")
skc.skc_pad_input(j.plan, x, xp, N)
y = j.forward_padded(xp)
for _ in range(2):
    j.forward_padded(xp, y)
torch.cuda.synchronize()
print("ok", layer, N)
