import os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tools')
import torch
import workloads as wl
from paper_1608_01409_b200 import skc
from sweep_regtile import time_conv
for cfg, li in [(2,1),(2,2),(2,3),(2,0),(4,0),(4,2)]:
    C = wl.CONFIGS[cfg]; L = C.layers[li]; N = C.batch
    w = wl.gen_weights(cfg, li, L)
    x = torch.from_numpy(wl.gen_input(cfg, li, L, 0, N)).cuda()
    for kb in ('', '110'):
        if kb: os.environ['SKC_DIRECT_SMEM_KB'] = kb
        else: os.environ.pop('SKC_DIRECT_SMEM_KB', None)
        conv = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups, skc.SKC_KERNEL_DIRECT)
        xp = torch.empty(conv.padded_shape(N), device='cuda'); skc.skc_pad_input(conv.plan, x, xp, N)
        out = torch.empty(conv.out_shape(N), device='cuda')
        ms = time_conv(conv, xp, out, N)
        g = conv.geom
        print(L.name, kb or 'auto', 'NS', g['stages'], 'smem', g['smem_bytes'], round(ms, 4), round(2*g['nnz']*L.Ho*L.Wo*N/ms/1e9, 2), flush=True)
