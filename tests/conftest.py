import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: takes more than ~20 s")


def reference_available() -> bool:
    return os.path.isdir(REFERENCE_SRC)


@pytest.fixture(scope="session")
def stmp_ref():
    """The unmodified reference package (build container only)."""
    if not reference_available():
        pytest.skip("reference not mounted (GPU box): covered by the golden fixtures")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import stmp
    return stmp


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def flat_from_fixture(z):
    from paper_1412_0680_b200 import tree as T
    return T._from_counts(
        tuple(int(k) for k in z["t_branching"]), int(z["t_n"]), int(z["t_fingerprint"][0]),
        _counts_by_depth(z), z["t_centroids"], z["t_leaf_atom"])


def _counts_by_depth(z):
    off = z["t_level_offsets"]
    cc = z["t_child_count"]
    return [cc[off[d]:off[d + 1]] for d in range(len(off) - 1)]
