import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: larger-scale cases")


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "results.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def gen_hashes():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "gen_hashes.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def datasets(tmp_path_factory):
    """Cache of generated datasets keyed by spec, written by the oracle generator (tests only)."""
    import oracle
    cache = {}
    base = tmp_path_factory.mktemp("data")

    def get(scale, nodes, devices, seed=42, codec="identity", rg_bytes=1 << 20):
        key = (scale, nodes, devices, seed, codec, rg_bytes)
        if key not in cache:
            d = str(base / ("d%d" % len(cache)))
            oracle.gen_tpch(d, scale, nodes, devices, seed, codec, rg_bytes)
            cache[key] = d
        return cache[key]

    return get
