"""Shared fixtures. `-m "not gpu"` runs everywhere (oracle vs golden, host logic, ABI load);
`-m gpu` needs a B200 and checks the CUDA path against the oracle and the reference goldens."""
from __future__ import annotations

import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA sm_100a (B200) device")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle

    if not oracle.ORACLE_SO.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "all"], check=True)
    return oracle.Oracle()


@pytest.fixture(scope="session")
def reference_lib():
    import oracle

    if not oracle.reference_available():
        pytest.skip("oracle/_ref (the compiled reference) is not built here")
    return oracle.Reference()


@pytest.fixture(scope="session")
def gold():
    cache = {}

    def load(name: str):
        if name not in cache:
            with np.load(GOLDEN / f"{name}.npz") as z:
                cache[name] = {k: z[k] for k in z.files}
        return cache[name]

    return load


def rel_err(a: np.ndarray, b: np.ndarray) -> tuple[float, float]:
    """(eps_inf, eps_2) of a against the reference b (SURVEY.md §8(c) parity definition)."""
    a = np.asarray(a)
    b = np.asarray(b)
    den_inf = float(np.max(np.abs(b))) if b.size else 0.0
    den_2 = float(np.linalg.norm(b.ravel()))
    num_inf = float(np.max(np.abs(a - b))) if b.size else 0.0
    num_2 = float(np.linalg.norm((a - b).ravel()))
    return (num_inf / den_inf if den_inf else num_inf, num_2 / den_2 if den_2 else num_2)
