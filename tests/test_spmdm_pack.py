"""Row f2, host side: the SpMDM kernel's tables (csrc/plan.cpp build_spmdm) decode back to the
canonical CSR (skc_plan_verify), the kernel is picked for FC plans by AUTO, and ineligible
geometries are refused.  No GPU needed: packing and verification are host-only."""
import numpy as np
import pytest

from paper_1608_01409_b200 import skc


def _fc(rng, M, K, density):
    return np.where(rng.random((M, K)) < density, rng.standard_normal((M, K)), 0).astype(np.float32)


@pytest.mark.parametrize("shape", [(1, 1, 4), (7, 13, 8), (40, 33, 64), (65, 100, 132),
                                   (300, 257, 256), (1000, 4096 // 8, 256), (33, 700, 12)])
def test_fc_plan_is_spmdm_and_verifies(shape):
    M, K, B = shape
    rng = np.random.default_rng(M * 7 + K)
    w = _fc(rng, M, K, 0.2)
    p = skc.skc_pack_fc(w, B)
    g = p.info()
    assert g["kernel"] == skc.SKC_KERNEL_SPMDM
    assert g["nnz"] == int(np.count_nonzero(w))
    assert g["pixels_per_lane"] in (4, 8) and g["channels_per_warp"] in (4, 8)
    assert g["smem_bytes"] <= 227 << 10
    skc.skc_plan_verify(p)


def test_fc_plan_edge_weights():
    """Empty rows, an all-zero matrix, a single dense row, a dense column."""
    rng = np.random.default_rng(3)
    w = _fc(rng, 50, 90, 0.1)
    w[5:9] = 0
    w[20] = rng.standard_normal(90)
    w[:, 17] = rng.standard_normal(50)
    for ww in (w, np.zeros((9, 31), np.float32)):
        p = skc.skc_pack_fc(ww, 64)
        assert p.info()["kernel"] == skc.SKC_KERNEL_SPMDM
        skc.skc_plan_verify(p)


def test_fc_odd_batch_falls_back_to_direct():
    rng = np.random.default_rng(4)
    w = _fc(rng, 20, 30, 0.3)
    assert skc.skc_pack_fc(w, 31).info()["kernel"] == skc.SKC_KERNEL_DIRECT
    with pytest.raises(skc.SkcError):
        skc.skc_pack_fc(w, 31, skc.SKC_KERNEL_SPMDM)


def test_spmdm_on_1x1_conv_plans():
    rng = np.random.default_rng(5)
    w = np.where(rng.random((24, 16, 1, 1)) < 0.3, rng.standard_normal((24, 16, 1, 1)), 0).astype(np.float32)
    p = skc.skc_pack_csr(w, 14, 14, 1, 0, 1, skc.SKC_KERNEL_SPMDM)
    assert p.info()["kernel"] == skc.SKC_KERNEL_SPMDM
    skc.skc_plan_verify(p)
    # ineligible: 3x3, stride 2, padding, groups, plane % 4 != 0
    w3 = rng.standard_normal((8, 4, 3, 3)).astype(np.float32)
    for args in [(w3, 9, 9, 1, 1, 1), (w[:, :, :, :], 14, 14, 2, 0, 1), (w, 14, 14, 1, 1, 1),
                 (w[:, :8], 14, 14, 1, 0, 2), (w, 7, 7, 1, 0, 1)]:
        with pytest.raises(skc.SkcError):
            skc.skc_pack_csr(*args, kernel=skc.SKC_KERNEL_SPMDM)


def test_spmdm_random_geometries_verify():
    rng = np.random.default_rng(6)
    for _ in range(60):
        M = int(rng.integers(1, 400))
        K = int(rng.integers(1, 1500))
        B = 4 * int(rng.integers(1, 150))
        w = _fc(rng, M, K, float(rng.choice([0.02, 0.1, 0.5, 1.0])))
        p = skc.skc_pack_fc(w, B)
        assert p.info()["kernel"] == skc.SKC_KERNEL_SPMDM
        skc.skc_plan_verify(p)
