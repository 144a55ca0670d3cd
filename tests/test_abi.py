"""The C-ABI library loads on a CPU-only host and exports exactly what
include/kgdist_b200.h declares (no compute calls without a GPU)."""

import ctypes
import os
import re

import numpy as np

from paper_2201_02791_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "kgdist_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(kg_[a-z0-9_]+)\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    decl = declared_symbols()
    assert decl, "no declarations parsed"
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(_lib.exported_symbols()) == decl
    assert lib.kg_abi_version() == _lib.ABI_VERSION


def test_status_codes_map_to_reference_errors():
    from paper_2201_02791_b200 import errors
    assert errors.STATUS_ERRORS[1] is errors.ValidationError
    assert errors.STATUS_ERRORS[4] is errors.SamplingError
    assert errors.STATUS_ERRORS[5] is errors.NumericError
    assert errors.STATUS_ERRORS[6] is errors.ProtocolError


def test_host_pcg64_peek_matches_numpy_raw_stream():
    gen = np.random.default_rng(2024)
    st = _lib.pcg_from_numpy(gen)
    out = np.zeros(16, dtype=np.uint64)
    _lib.load().kg_pcg64_peek64(ctypes.byref(st), out.ctypes.data, 16)
    np.testing.assert_array_equal(out, gen.bit_generator.random_raw(16))


def test_compute_path_fails_loudly_without_cuda():
    import pytest
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2201_02791_b200 import errors
    with pytest.raises(errors.DeviceError):
        _lib.require_cuda()


def test_host_consume32_matches_numpy_for_every_parity():
    for seed in range(6):
        for pre in (0, 1):
            for count in (1, 2, 3, 4, 9, 10):
                gen = np.random.default_rng(seed)
                if pre:
                    gen.integers(0, 2 ** 32, size=1, dtype=np.uint32)   # leave a buffered half
                st = _lib.pcg_from_numpy(gen)
                gen.integers(0, 2 ** 32, size=count, dtype=np.uint32)
                _lib.pcg_consume32(st, count)
                s = gen.bit_generator.state
                assert ((st.state_hi << 64) | st.state_lo) == s["state"]["state"]
                assert (st.has_uint32, st.uinteger) == (s["has_uint32"], s["uinteger"])
