import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def golden(name):
    return os.path.join(ROOT, "tests", "golden", name)


def read_sections(path):
    """Parse a golden file of '# comments', section names and integer/float rows."""
    import numpy as np
    out, cur = {}, None
    for line in open(path):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        toks = line.split()
        if len(toks) == 1 and toks[0].isalpha():
            cur = toks[0]
            out[cur] = []
        else:
            out.setdefault(cur, []).append([float(t) for t in toks])
    return {k: np.array(v) for k, v in out.items()}


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


def relF(x, ref):
    import numpy as np
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(x - ref) / (den if den > 0 else 1.0))
