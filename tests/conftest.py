import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


_GPU_SELECTED = False


def pytest_collection_modifyitems(session, config, items):
    global _GPU_SELECTED
    _GPU_SELECTED = any(item.get_closest_marker("gpu") for item in items)


@pytest.fixture(scope="session", autouse=True)
def _warm_jit_cache():
    """GPU sessions: compile the JIT code of every BASELINE config layer up front, in
    parallel host threads (whole-program compiles are serial per plan, 20-45 s each), into the
    on-disk cache the tests' own plans then hit -- the same weights give the same code.  Pure
    host work (no GPU); skipped for CPU-only sessions."""
    if not _GPU_SELECTED:
        yield
        return
    try:
        import torch
        if not torch.cuda.is_available():
            yield
            return
        import concurrent.futures as cf
        import workloads as wl
        from paper_1608_01409_b200 import skc
        skc.lib()
        plans = []
        for cfg_id in (1, 2, 3, 4, 5):
            cfg = wl.CONFIGS[cfg_id]
            for li, L in enumerate(cfg.layers):
                try:
                    plans.append(skc.skc_pack_csr(wl.gen_weights(cfg_id, li, L), L.H, L.W, L.stride,
                                                  L.pad, L.groups, skc.SKC_KERNEL_AUTO))
                except skc.SkcError:
                    pass
        with cf.ThreadPoolExecutor(max_workers=max(1, min(len(plans), os.cpu_count() or 4))) as ex:
            list(ex.map(lambda p: skc.skc_plan_compile(p), plans))
    except Exception:  # noqa: BLE001 -- warming is an optimisation only
        pass
    yield
