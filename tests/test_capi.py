"""The C-ABI library: loads, exports include/rmfht.h, validates like the
reference, expands maps like the oracle.  No GPU compute here."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2108_12550_b200 import _native
from paper_2108_12550_b200.automorphism import random_raw_table
from paper_2108_12550_b200.plan import map_sizes


def _declared():
    src = open(os.path.join(ROOT, "include", "rmfht.h")).read()
    return sorted(set(re.findall(r"\b(rmfht_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    declared = _declared()
    assert set(declared) == set(_native.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.rmfht_version() >= 1


def _create(r, m, L, M, flags=1, dtype=0):
    lib = _native.lib()
    h = ctypes.c_void_p()
    rc = lib.rmfht_plan_create(r, m, L, M, flags, dtype, ctypes.byref(h))
    return rc, h


@pytest.mark.parametrize("r,m,L,M,code", [(0, 5, 1, 1, -1), (5, 5, 1, 1, -1), (2, 15, 1, 1, -1),
                                          (2, 9, 0, 1, -1), (2, 9, 4, 0, -1), (2, 12, 4, 5, -3)])
def test_plan_create_errors(r, m, L, M, code):
    rc, h = _create(r, m, L, M)
    assert rc == code and not h.value
    assert _native.last_error()


def test_plan_layout_matches_host_schedule():
    lib = _native.lib()
    for (r, m, L, M) in [(2, 9, 4, 20), (3, 7, 8, 32), (2, 9, 1, 512), (2, 7, 2, 4)]:
        rc, h = _create(r, m, L, M)
        assert rc == 0, _native.last_error()
        S = lib.rmfht_plan_maps_per_attempt(h)
        sizes = (ctypes.c_int * S)()
        lib.rmfht_plan_map_sizes(h, sizes)
        assert list(sizes) == map_sizes(r, m, L)
        assert lib.rmfht_plan_record_u16(h) == 2 * m + 2
        lib.rmfht_plan_destroy(h)


def test_expand_maps_matches_oracle(oracle_mod):
    lib = _native.lib()
    r, m, L = 3, 7, 8
    rc, h = _create(r, m, L, 4)
    sizes = map_sizes(r, m, L)
    raw = random_raw_table(np.random.default_rng(3), (3, 4), sizes, m)
    rec = np.zeros(raw.shape[:-1] + (2 * m + 2,), dtype=np.uint16)
    assert lib.rmfht_expand_maps(h, raw.ctypes.data, rec.ctypes.data, raw.size // (m + 1)) == 0
    rec2 = np.zeros_like(rec)
    sz = np.asarray(sizes, dtype=np.int32)
    assert oracle_mod.lib().rmo_expand_table(raw.ctypes.data, raw.size // (m + 1), m, sz.ctypes.data,
                                              len(sizes), rec2.ctypes.data) == 0
    assert np.array_equal(rec, rec2)
    # a singular map is a ValueError-class error
    raw[1, 2, 5, :] = 0
    assert lib.rmfht_expand_maps(h, raw.ctypes.data, rec.ctypes.data, raw.size // (m + 1)) == -2
    assert "invertible" in _native.last_error()
    lib.rmfht_plan_destroy(h)


def test_uncompiled_shape_binds_generic_kernel():
    lib = _native.lib()
    rc, h = _create(2, 9, 3, 5)
    assert rc == 0 and lib.rmfht_plan_kernel(h) == 3
    lib.rmfht_plan_destroy(h)
    rc, h = _create(2, 9, 4, 20)
    assert rc == 0 and lib.rmfht_plan_kernel(h) == 2
    lib.rmfht_plan_destroy(h)
    rc, h = _create(2, 9, 4, 20, 1, 1)
    assert rc == 0 and lib.rmfht_plan_kernel(h) == 1
    lib.rmfht_plan_destroy(h)
    # the specialised float32 kernels of the BASELINE shapes: pair kernel
    # (r = 2, L = 2, M | 16), lane-group kernel (r = 2, L = 1, 4 | M)
    for (r, m, L, M, kid) in [(2, 7, 2, 4, 6), (2, 7, 2, 3, 2), (2, 9, 1, 512, 7), (2, 9, 1, 6, 2)]:
        rc, h = _create(r, m, L, M)
        assert rc == 0 and lib.rmfht_plan_kernel(h) == kid, (r, m, L, M)
        lib.rmfht_plan_destroy(h)


def test_workspace_bytes_contract():
    """Caller-owned workspace (rmfht_workspace_bytes): the throughput kernel
    needs per-attempt records, sampled launches the table too; the float64
    kernel needs none; bad batches are ValueError-class."""
    lib = _native.lib()
    rc, h = _create(2, 9, 4, 20)
    w0 = lib.rmfht_workspace_bytes(h, 1000, 0)
    w1 = lib.rmfht_workspace_bytes(h, 1000, 1)
    assert 1000 * 20 * (16 + 8 * 8) <= w0 < w1
    assert w1 - w0 >= 1000 * 20 * 12 * 40
    assert w0 % 256 == 0 and w1 % 256 == 0
    assert lib.rmfht_workspace_bytes(h, 0, 1) == 0
    assert lib.rmfht_workspace_bytes(h, -1, 0) == -2
    lib.rmfht_plan_destroy(h)
    rc, h = _create(2, 9, 4, 20, 1, 1)
    assert lib.rmfht_workspace_bytes(h, 1000, 0) == 0
    assert lib.rmfht_workspace_bytes(h, 1000, 1) == 1000 * 20 * 12 * 40
    lib.rmfht_plan_destroy(h)


def test_workspace_bytes_contract():
    """Caller-owned workspace (rmfht_workspace_bytes): the throughput kernel
    needs per-attempt records, sampled launches the table too; the float64
    kernel needs none; bad batches are ValueError-class."""
    lib = _native.lib()
    rc, h = _create(2, 9, 4, 20)
    w0 = lib.rmfht_workspace_bytes(h, 1000, 0)
    w1 = lib.rmfht_workspace_bytes(h, 1000, 1)
    assert 1000 * 20 * (16 + 8 * 8) <= w0 < w1
    assert w1 - w0 >= 1000 * 20 * 12 * 40
    assert w0 % 256 == 0 and w1 % 256 == 0
    assert lib.rmfht_workspace_bytes(h, 0, 1) == 0
    assert lib.rmfht_workspace_bytes(h, -1, 0) == -2
    lib.rmfht_plan_destroy(h)
    rc, h = _create(2, 9, 4, 20, 1, 1)
    assert lib.rmfht_workspace_bytes(h, 1000, 0) == 0
    assert lib.rmfht_workspace_bytes(h, 1000, 1) == 1000 * 20 * 12 * 40
    lib.rmfht_plan_destroy(h)


def test_unsupported_shape_is_a_configuration_error():
    """RMFHT_EUNSUPPORTED surfaces as top_decoders.UnsupportedShape, a
    ConfigurationError subclass the INTEGRATION.md binding falls back on."""
    from paper_2108_12550_b200.decoder import Plan
    from paper_2108_12550_b200.rm_core import ConfigurationError
    from paper_2108_12550_b200.top_decoders import UnsupportedShape
    assert issubclass(UnsupportedShape, ConfigurationError)
    with pytest.raises(UnsupportedShape):
        Plan(2, 12, 4, 5)
    with pytest.raises(ConfigurationError) as e:
        Plan(2, 15, 4, 5)
    assert not isinstance(e.value, UnsupportedShape)
