import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle
    try:
        return oracle.Reference()
    except FileNotFoundError as e:
        pytest.skip(str(e))


def load_corpus():
    z = np.load(os.path.join(GOLDEN, "corpus.npz"))
    imgs, off = [], 0
    for h, w in z["shapes"]:
        n = int(h) * int(w)
        imgs.append(z["pixels"][off:off + n].reshape(int(h), int(w)))
        off += n
    return imgs, z


def load_selection():
    return np.load(os.path.join(GOLDEN, "selection.npz"))


@pytest.fixture(scope="session")
def corpus():
    return load_corpus()


@pytest.fixture(scope="session")
def selection():
    return load_selection()


@pytest.fixture(scope="session")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test requested but no CUDA device is visible")
    from paper_1707_05062_b200 import default_context
    return default_context()
