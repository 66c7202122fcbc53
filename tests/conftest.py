import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size) case")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def tiny_golden():
    return load_golden("tiny")


@pytest.fixture(scope="session")
def small_golden():
    return load_golden("small")


def small_case(g, seed):
    p = f"c{seed}_"
    meta = g[p + "meta"]
    U, I, nnz, d, b = (int(x) for x in meta[:5])
    a0, reg, nu = (float(x) for x in meta[5:])
    case = {k[len(p):]: v for k, v in g.items() if k.startswith(p)}
    case.update(U=U, I=I, nnz=nnz, d=d, b=b, alpha0=a0, reg=reg, nu=nu)
    if "partition" in case:
        arr = list(case["partition"])
        cut = arr.index(-1)
        flat, sizes = arr[:cut], arr[cut + 1:]
        blocks, s = [], 0
        for n in sizes:
            blocks.append(np.array(flat[s:s + n]))
            s += n
        case["blocks"] = blocks
    return case


def relf(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def relmax(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))
