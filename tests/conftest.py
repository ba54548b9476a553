import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: longer statistical tests")


def load_golden(name: str) -> dict:
    g = np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
    d = {k: g[k] for k in g.files}
    d["config"] = json.loads(str(d["config"]))
    d["scene"] = str(d["scene"])
    d["dump"] = str(d["dump"])
    return d


STAT_KEYS = ["b", "b_stderr", "total_mutations", "perturbation_proposals", "large_step_proposals",
             "mean_acceptance", "film_luminance", "identity_residual", "region_count",
             "rays_closest", "rays_visibility"]


def golden_stats(d: dict) -> dict:
    return dict(zip(STAT_KEYS, d["stats"].tolist()))


GOLDEN_CASES = sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz"))


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle.abi import OracleLib, ORACLE_SO, build
    if not os.path.exists(ORACLE_SO):
        build(reference=False)
    return OracleLib()


@pytest.fixture(scope="session")
def ref_lib():
    from oracle.abi import RefLib, REF_LOG_SO
    if not os.path.exists(REF_LOG_SO):
        pytest.skip("reference harness not built (needs /root/reference at build time)")
    return RefLib(log=True)


def has_gpu() -> bool:
    import ctypes
    try:
        cuda = ctypes.CDLL("libcuda.so.1")
        if cuda.cuInit(0) != 0:
            return False
        n = ctypes.c_int()
        return cuda.cuDeviceGetCount(ctypes.byref(n)) == 0 and n.value > 0
    except OSError:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
