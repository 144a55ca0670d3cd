"""Shared pytest setup: the `gpu` marker, fixture loaders and import paths.

`-m "not gpu"` tests run on the CPU-only container (oracle vs golden
fixtures, host logic, C-ABI symbol checks); `-m gpu` tests need a B200 and
call the CUDA path through the C ABI.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


def golden_json(g: dict, key: str = "config_json") -> dict:
    import json
    return json.loads(bytes(g[key]).decode())


def rng_from_state(arr) -> np.random.Generator:
    """numpy Generator positioned at a state captured by make_golden.rng_state."""
    a = [int(x) for x in arr]
    g = np.random.default_rng(0)
    g.bit_generator.state = {
        "bit_generator": "PCG64",
        "state": {"state": (a[0] << 64) | a[1], "inc": (a[2] << 64) | a[3]},
        "has_uint32": a[4], "uinteger": a[5]}
    return g


def state_tuple(gen) -> tuple:
    st = gen.bit_generator.state
    return (st["state"]["state"], st["state"]["inc"], st["has_uint32"], st["uinteger"])


@pytest.fixture(scope="session")
def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
