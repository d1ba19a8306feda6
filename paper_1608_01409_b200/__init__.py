"""paper_1608_01409_b200 -- B200-native direct sparse convolution (arXiv:1608.01409).

The hot path lives in libskc.so (csrc/, C-ABI in include/skc.h); `skc` is its ctypes
binding.  Importing this package does not touch the GPU; calling into libskc raises if the
library was not built (there is no CPU fallback).
"""
from . import skc  # noqa: F401
from .skc import (SKC_KERNEL_AUTO, SKC_KERNEL_DIRECT, SKC_KERNEL_REGTILE, Plan,  # noqa: F401
                  SkcError, SparseConv2d, skc_forward_host, skc_layout_offset,
                  skc_model_layer_cost, skc_model_project, skc_model_window, skc_pack_csr,
                  skc_pad_input, skc_plan_upload, skc_sparse_conv_forward)
