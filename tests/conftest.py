import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _ensure_built():
    """Builds the checkers (C oracle, host build of the engine source) and
    the product library if a fresh checkout lacks them (nvcc cross-compiles
    without a GPU). On the GPU box the prebuilt files travel with the repo."""
    import subprocess
    need_checkers = not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")) or \
        not os.path.exists(os.path.join(ROOT, "tests", "_hostsim", "libeconoserve_hostsim.so"))
    need_product = not os.path.exists(os.path.join(ROOT, "paper_2411_06364_b200", "_lib",
                                                   "libeconoserve_b200.so"))
    if need_checkers or need_product:
        import __graft_entry__ as ge
        try:
            if need_checkers:
                ge.build_checkers()
            if need_product:
                ge.build_product()
        except (subprocess.CalledProcessError, FileNotFoundError) as ex:
            print("build of test artefacts failed:", ex)


_ensure_built()

HOSTSIM = os.path.join(ROOT, "tests", "_hostsim", "libeconoserve_hostsim.so")


def make_engine(backend, trace, opts):
    """Engine factory over the three implementations that share one API:
    'oracle' (C restatement), 'hostsim' (the product engine source compiled
    for the host, test-only) and 'device' (the sm_100a product)."""
    if backend == "oracle":
        from oracle import port
        return port.OracleEngine(trace, opts)
    from paper_2411_06364_b200.engine import Engine
    if backend == "hostsim":
        return Engine(trace, opts, lib=HOSTSIM)
    return Engine(trace, opts)


BACKENDS = ["oracle", "hostsim", pytest.param("device", marks=pytest.mark.gpu)]
