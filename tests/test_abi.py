"""The C-ABI boundary (include/slsht_cuda.h) without a GPU: the product library loads, exports
every declared entry point, and validates arguments with the reference's error convention
before touching a device; the product path never imports the oracle."""
from __future__ import annotations

import ctypes as C
import re
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_functions() -> list[str]:
    text = (ROOT / "include" / "slsht_cuda.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(slsht_cuda_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import paper_1207_5558_b200 as S

    lib = S.load()
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    from paper_1207_5558_b200 import _lib

    assert sorted(_lib.EXPORTS) == names


def test_library_is_sm100a_only():
    lib = ROOT / "paper_1207_5558_b200" / "libslsht_cuda.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_\d+a?", out.stdout))
    assert arches == {"sm_100a"}, arches


def test_dmma_in_sass():
    lib = ROOT / "paper_1207_5558_b200" / "libslsht_cuda.so"
    out = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "DMMA.8x8x4" in out.stdout  # FP64 tensor-core tiles in the coupling/modulated GEMMs


def _cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def test_validation_precedes_device_checks():
    import paper_1207_5558_b200 as S

    # lmax > L_f + L_h -> ValidationError (transform.cpp:250-252) even without a GPU
    with pytest.raises(S.ValidationError, match="L_f \\+ L_h"):
        S.Plan(4, 2, lmax=7)
    with pytest.raises(S.ValidationError):
        S.Plan(-1, 2)
    with pytest.raises(S.ValidationError):
        S.SphCoeffs(3, np.zeros(5))
    f = S.SphCoeffs(3, np.zeros(16))
    h = S.SphCoeffs(1, np.zeros(4))
    with pytest.raises(S.ValidationError):
        S.forward_fast(f, h, opts=S.ForwardOptions(lmax=5))
    with pytest.raises(S.ValidationError):  # arguments are checked before the device
        S.forward_direct(S.SphCoeffs(2, np.zeros(9)), S.SphCoeffs(3, np.zeros(16)), cells=[])


@pytest.mark.skipif(_cuda_available(), reason="checks the no-GPU error path")
def test_no_cpu_fallback_without_gpu():
    import paper_1207_5558_b200 as S

    with pytest.raises(S.DeviceError, match="no CPU fallback"):
        S.Plan(4, 2)
    with pytest.raises(S.DeviceError):
        S.delta_tables(4)
    with pytest.raises(S.DeviceError, match="no CPU fallback"):  # the direct engine too
        S.forward_direct(S.SphCoeffs(2, np.zeros(9)), S.SphCoeffs(1, np.zeros(4)))


def test_product_never_imports_the_oracle():
    code = ("import sys; sys.path.insert(0, %r); import paper_1207_5558_b200 as S; "
            "import paper_1207_5558_b200.configs, paper_1207_5558_b200.parallel; "
            "assert 'oracle' not in sys.modules, sorted(sys.modules)" % str(ROOT))
    subprocess.run([sys.executable, "-c", code], check=True)


def test_digest_weight_bit_trick_is_exact():
    # kernels_couple.cuh digest_weight: (2^52 + x) * 2^-24 - (2^28 + 1/2) == x * 2^-24 - 1/2
    rng = np.random.default_rng(3)
    x = rng.integers(0, 1 << 24, 100000, dtype=np.uint64)
    d = (np.uint64(0x43300000) << np.uint64(32)) | x
    dd = d.view(np.float64)
    got = dd * (1.0 / 16777216.0) - (268435456.0 + 0.5)
    assert np.array_equal(got, x.astype(np.float64) * 2.0 ** -24 - 0.5)
