import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def read_golden(name):
    """Parse a golden fixture: '#' comments, then 'key v1 v2 ...' lines (ints auto-detect hex)."""
    out = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            key, *vals = line.split()
            conv = []
            for v in vals:
                if v.lower().startswith("0x"):
                    conv.append(int(v, 16))
                elif "." in v or "e" in v.lower():
                    conv.append(float(v))
                else:
                    conv.append(int(v))
            out.setdefault(key, []).append(conv)
    return out


@pytest.fixture(scope="session")
def golden():
    return read_golden


@pytest.fixture(scope="session")
def paper():
    from oracle import oracle as O
    return O.default_params()
