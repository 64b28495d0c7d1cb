import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden_v1.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; parity tests proper")


@pytest.fixture(scope="session")
def oracle_c():
    from oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle import REF_SO, Reference

    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return Reference()


class Golden:
    def __init__(self, path):
        self.z = np.load(path)
        self.names = [str(n) for n in self.z["__names__"]]

    def case(self, name):
        g = {k.split("/", 1)[1]: self.z[k] for k in self.z.files if k.startswith(name + "/")}
        for key in ("q", "k", "v", "meta_min", "meta_max"):
            g[key] = g[key].astype(np.float32)
        g["S"] = int(g["S"])
        return g


@pytest.fixture(scope="session")
def golden():
    return Golden(GOLDEN)


def half(a):
    """Round to fp16 (RNE) and widen back to float32: the values the GPU and the
    reference both see."""
    return np.asarray(a, dtype=np.float32).astype(np.float16).astype(np.float32)
