import os, sys, json
sys.path.insert(0, '.')
import torch
import workloads as wl
from paper_1608_01409_b200 import skc
sys.path.insert(0, 'tools')
from sweep_regtile import time_conv
for cfg, li in [(2,1),(2,2),(2,3),(3,7),(3,6),(2,0),(4,0),(4,3)]:
    C = wl.CONFIGS[cfg]; L = C.layers[li]; N = C.batch
    w = wl.gen_weights(cfg, li, L)
    x = torch.from_numpy(wl.gen_input(cfg, li, L, 0, N)).cuda()
    for nw, m in [(8,2),(16,2),(8,4),(16,4),(12,2),(12,4),(8,1),(16,1)]:
        os.environ['SKC_DIRECT_NW'] = str(nw); os.environ['SKC_DIRECT_M'] = str(m)
        try:
            conv = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups, skc.SKC_KERNEL_DIRECT)
        except Exception as e:
            print(L.name, nw, m, e); continue
        xp = torch.empty(conv.padded_shape(N), device='cuda'); skc.skc_pad_input(conv.plan, x, xp, N)
        out = torch.empty(conv.out_shape(N), device='cuda')
        ms = time_conv(conv, xp, out, N)
        g = conv.geom
        print(json.dumps(dict(layer=L.name, nw=nw, m=g['channels_per_warp'], T=g['pixels_per_lane'], ni=g['images_per_cta'], cb=g['chunk_channels'], ns=g['stages'], smem=g['smem_bytes'], ms=round(ms,4), tf=round(2*g['nnz']*L.Ho*L.Wo*N/ms/1e9,2))), flush=True)
