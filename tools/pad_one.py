"""Run skc_pad_input for one AlexNet layer of config 2 (JIT plan, pair layout) a few times (for ncu)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1608_01409_b200 import skc  # noqa: E402
import workloads as wl  # noqa: E402
layer, N = sys.argv[1], int(sys.argv[2])
cfg = wl.CONFIGS[2]
li = [L.name for L in cfg.layers].index(layer)
L = cfg.layers[li]
w = wl.gen_weights(2, li, L)
x = torch.from_numpy(wl.gen_input(2, li, L, 0, N)).cuda()
p = skc.skc_pack_csr(w, L.H, L.W, L.stride, L.pad, L.groups, skc.SKC_KERNEL_JIT)
xp = torch.empty(skc.padded_shape(p.info(), N), device="cuda")
for _ in range(3):
    skc.skc_pad_input(p, x, xp, N)
torch.cuda.synchronize()
print("ok", layer, N)
