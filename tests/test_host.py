"""CPU tests: the C ABI library loads and exports every declared symbol, and
the host-side logic (grid, problems, hierarchy shapes) matches the reference
(golden fixtures / reference test expectations)."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "helmfree_b200.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(hf_[a-z_0-9]+)\s*\(", text)))


def test_header_symbols_match_binding_list():
    from paper_2308_06085_b200 import _native
    assert _declared_symbols() == sorted(_native.EXPORTED)


def test_library_loads_and_exports_every_symbol():
    from paper_2308_06085_b200 import _native, build_native
    build_native.build()
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in _declared_symbols():
        assert hasattr(lib, name), name
    L = _native.load()
    assert L.hf_version() == 2


def test_missing_library_fails_loudly(tmp_path):
    from paper_2308_06085_b200 import _native
    with pytest.raises(_native.NativeUnavailable):
        _native._lib_backup = _native._lib
        try:
            _native._lib = None
            _native.load(str(tmp_path / "nope.so"))
        finally:
            _native._lib = _native._lib_backup


class TestGrid:
    def test_coarsen_trace_salt(self):
        from paper_2308_06085_b200.grid import make_grid
        from paper_2308_06085_b200.multigrid import MGConfig, keep_coarsening
        from paper_2308_06085_b200.grid import coarsen
        g = make_grid(641, 641, 193, 20.0)
        while keep_coarsening(g, MGConfig()):
            g = coarsen(g)
        assert g.shape == (41, 41, 13)

    def test_not_coarsenable(self):
        from paper_2308_06085_b200.grid import NotCoarsenable, coarsen, make_grid
        with pytest.raises(NotCoarsenable):
            coarsen(make_grid(4, 5, 5, 1.0))

    def test_dimension_too_small(self):
        from paper_2308_06085_b200.grid import DimensionTooSmall, make_grid
        with pytest.raises(DimensionTooSmall):
            make_grid(2, 5, 5, 1.0)

    def test_global_local_round_trip(self):
        from paper_2308_06085_b200.grid import BlockExtent, global_to_local, local_to_global
        e = BlockExtent(33, 1, 1, 65, 65, 65)
        assert global_to_local(e, (33, 1, 1)) == (1, 1, 1)
        assert global_to_local(e, (32, 5, 5)) is None
        assert local_to_global(e, global_to_local(e, (40, 7, 9))) == (40, 7, 9)


@pytest.mark.filterwarnings("ignore:kh =")
class TestProblems:
    def test_closed_off_rhs_matches_reference(self):
        from paper_2308_06085_b200 import problems
        gold = np.load(os.path.join(GOLD, "problems.npz"))
        p = problems.closed_off_problem(9, 10.0)
        _, b = problems.build_problem(p)
        np.testing.assert_allclose(b, gold["closed_off_9_k10_rhs"], rtol=1e-14, atol=1e-12)

    def test_wedge_medium_and_dirac_match_reference(self):
        from paper_2308_06085_b200 import problems
        gold = np.load(os.path.join(GOLD, "problems.npz"))
        w = problems.wedge_problem(shape=(13, 13, 21))
        spec, b = problems.build_problem(w)
        np.testing.assert_array_equal(spec.k_field, gold["wedge_13_k"])
        np.testing.assert_array_equal(b, gold["wedge_13_rhs"])

    def test_dirac_unit_integral(self):
        from paper_2308_06085_b200 import problems
        p = problems.point_source_cube(33, 20.0)
        _, b = problems.build_problem(p)
        assert np.sum(b) * p.grid.h ** 3 == 1.0

    def test_wedge3_geometry(self):
        from paper_2308_06085_b200 import problems
        from paper_2308_06085_b200.grid import full_extent
        p = problems.wedge3_problem(33)
        k = p.medium.k_field(p.grid, full_extent(p.grid))
        c = 2 * np.pi * p.medium.frequency / k
        # x = 0: top layer above z = 0.4, bottom layer below z = 0.8
        assert c[0, 0, 0] == 2000.0 and c[0, 0, 16] == 1500.0 and c[0, 0, 32] == 3000.0
        assert abs(np.max(k) * p.grid.h - problems.KH_LIMIT) < 1e-12

    def test_random_medium_band(self):
        from paper_2308_06085_b200 import problems
        v = problems.random_medium_velocity((33, 33, 17), seed=1)
        assert v.min() >= 1500.0 and v.max() <= 4500.0 and (v == 4500.0).any()
        np.testing.assert_array_equal(v, problems.random_medium_velocity((33, 33, 17), seed=1))

    def test_velocity_file_round_trip(self, tmp_path):
        from paper_2308_06085_b200 import problems
        path = tmp_path / "v.bin"
        c = problems.gen_salt_surrogate(path, (9, 9, 5))
        m = problems.read_velocity_grid(path, (9, 9, 5))
        np.testing.assert_array_equal(np.asarray(m.velocities), c)
        with pytest.raises(problems.ProblemError):
            problems.read_velocity_grid(path, (9, 9, 6))


def test_abi_argument_errors_without_a_gpu():
    """Argument validation of the C ABI runs before any CUDA call: bad handles
    and requests come back as error codes / NULL with a message."""
    import ctypes as C
    from paper_2308_06085_b200 import _native
    L = _native.load()
    assert not L.hf_bcg_create(None, 1e-6, 10, 1e-30)
    assert "Bi-CGSTAB state" in _native.last_error()
    ms = C.c_float()
    assert L.hf_solver_bench_vec(None, 0, 1, C.byref(ms)) == _native.ERR_ARG
    assert L.hf_bcg_step(None, 2, None) == _native.ERR_ARG
    assert L.hf_level_down_restrict(None, 0, None, None) == _native.ERR_ARG
    assert L.hf_level_up(None, 0, None, None, None) == _native.ERR_ARG


def test_kernel_variant_options_are_named_and_default_off():
    """Every kernel-variant option DESIGN.md section 9 lists is known to
    hf_set_option / hf_get_option, off by default, and unknown names are
    rejected (the library reads no environment variables)."""
    from paper_2308_06085_b200 import _native
    L = _native.load()
    names = ["no_pdl", "no_flat", "no_flat_dr", "no_dr", "tiled_dr", "flat_up", "fuse_up", "no_fuse",
             "coarsest_dense", "no_palette", "no_wide", "force_wide", "wide_p4", "wide_all",
             "no_wide_up", "wide_p3", "wide_p1", "wide_big"]
    for n in names:
        assert L.hf_get_option(n.encode()) == 0, n
        _native.set_option(n, 1)
        assert L.hf_get_option(n.encode()) == 1
        _native.set_option(n, 0)
    assert L.hf_get_option(b"no_such_option") == _native.ERR_ARG
    with pytest.raises(_native.NativeError):
        _native.set_option("no_such_option", 1)
