"""C-ABI contract checks that need no GPU (-m "not gpu"): the library builds and loads,
exports every symbol include/duquad.h declares, host-only helpers work, and device
calls fail loudly (status, not crash) without a device."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1504_05708_b200 import build, _lib
    build.build()
    return _lib.load()


def _header_functions():
    src = open(os.path.join(ROOT, "include", "duquad.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(duquad_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = _header_functions()
    assert "duquad_solve" in names and "duquad_setup" in names and "duquad_lipschitz" in names
    for name in names:
        assert hasattr(lib, name), name
    from paper_1504_05708_b200 import _lib
    assert set(_lib.EXPORTED) == set(names)


def test_abi_version_and_status_strings(lib):
    assert lib.duquad_abi_version() == 4
    assert lib.duquad_status_string(0) == b"ok"
    assert b"invalid" in lib.duquad_status_string(1)


def test_default_options(lib):
    from paper_1504_05708_b200 import _lib
    o = _lib.Options()
    lib.duquad_default_options(C.byref(o))
    assert o.dual_step_scale == 0.5 and o.project_dual == 1 and o.world_size == 1 and o.use_graphs == 1
    assert o.sell_path == 1 and o.pair_rows == 1 and o.pdl == 1 and o.fused_path == 1 and o.nccl_self == 0


def test_ctypes_mirrors_match_the_abi_structs(lib):
    """Every ctypes mirror of an ABI struct has the C struct's size (a field added on one side only
    would shift every later field)."""
    from paper_1504_05708_b200 import _lib
    for which, cls in enumerate((_lib.Problem, _lib.Options, _lib.Result, _lib.Schedule, _lib.Bounds, _lib.Monitor)):
        assert lib.duquad_struct_size(which) == C.sizeof(cls), cls.__name__
    assert lib.duquad_struct_size(99) == -1


@pytest.mark.parametrize("rows,world", [(16384, 8), (10, 3), (5, 8), (0, 2), (2000, 1)])
def test_shard_range_partitions(lib, rows, world):
    from paper_1504_05708_b200 import shard_range
    covered = []
    for r in range(world):
        b, e = shard_range(rows, world, r)
        assert 0 <= b <= e <= rows
        covered.extend(range(b, e))
    assert covered == list(range(rows))


def test_shard_range_rejects_bad_args(lib):
    b, e = C.c_int64(), C.c_int64()
    assert lib.duquad_shard_range(10, 2, 2, C.byref(b), C.byref(e)) == 1
    assert lib.duquad_shard_range(10, 0, 0, C.byref(b), C.byref(e)) == 1


def test_setup_validation_errors_without_device(lib):
    """Argument errors are reported before any device call; with valid args and no GPU the
    status is ENODEV (never a silent CPU fallback)."""
    import numpy as np
    from paper_1504_05708_b200 import _lib
    n, p = 4, 2
    Q = np.eye(n)
    G = np.ones((p, n))
    q, g, lb, ub = np.zeros(n), np.zeros(p), -np.ones(n), np.ones(n)
    prob = _lib.Problem()
    prob.n, prob.p, prob.batch, prob.format, prob.on_device = n, p, 1, 0, 0
    prob.Q, prob.ldQ, prob.G, prob.ldG = Q.ctypes.data, n, G.ctypes.data, n
    prob.q, prob.g, prob.lb, prob.ub = q.ctypes.data, g.ctypes.data, lb.ctypes.data, ub.ctypes.data
    prob.cone, prob.cone_all = None, 1
    ctx = C.c_void_p()
    assert lib.duquad_setup(C.byref(ctx), C.byref(prob), -1.0, None) == _lib.DUQUAD_EINVAL   # rho < 0
    bad_ub = np.array([1.0, 1.0, -2.0, 1.0])
    prob.ub = bad_ub.ctypes.data
    assert lib.duquad_setup(C.byref(ctx), C.byref(prob), 1.0, None) == _lib.DUQUAD_EINVAL    # lb > ub
    assert b"lb <= ub" in lib.duquad_last_error(None)
    prob.ub = ub.ctypes.data
    Qn = Q.copy()
    Qn[1, 2] = float("nan")
    prob.Q = Qn.ctypes.data
    assert lib.duquad_setup(C.byref(ctx), C.byref(prob), 1.0, None) == _lib.DUQUAD_EINVAL    # NaN
    prob.Q = Q.ctypes.data
    import torch
    if not torch.cuda.is_available():
        assert lib.duquad_setup(C.byref(ctx), C.byref(prob), 1.0, None) == _lib.DUQUAD_ENODEV
        assert not ctx.value


def test_product_package_does_not_touch_oracle():
    """The product path never imports the oracle (no CPU fallback route)."""
    pkg = os.path.join(ROOT, "paper_1504_05708_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in txt.replace("oracle/", "").lower() or f == "__init__.py", f
                assert "import oracle" not in txt and "from oracle" not in txt, f


def test_theory_schedule_host_only(lib):
    """duquad_theory_schedule is host arithmetic (no device): the same numbers as the oracle's
    theory_schedule (which tests/test_oracle_pins.py pins to Theorem 1 and Lemma 1)."""
    from oracle import dfom as O
    from paper_1504_05708_b200 import theory_schedule, _lib
    for alg in ("DGM", "DFGM"):
        for args in [(1e-2, 1.0, 1.0, 40.0, 0.5, 2.0, 3.0, 0.1, 2.0), (1e-3, 3.7, 0.25, 1e4, 0.0, 1.0, 7.0, 0.0, 0.0),
                     (0.5, 12.0, 40.0, 9.0, 1e-3, 2.0, 1.5, 0.0, 5.0), (1e-2, 1.0, 1.0, 40.0, 0.5, 2.0, 0.0, 1e-12, 1.0),
                     (1e-2, 1.0, 1.0, 40.0, 0.5, 2.0, 3.0, 2e-7, 1.0), (1e-2, 1.0, 1.0, 40.0, 0.5, 2.0, 3.0, 2e-7, 3.0)]:
            got = theory_schedule(alg, *args)
            want = O.theory_schedule(alg, *args[:7], lambda_min_Q=args[7], lambda_max_Q=args[8])
            for k in ("k_out", "k_in", "k_total", "case_id"):
                assert got[k] == want[k], (alg, args, k)
            for k in ("eps_in", "rho_star"):
                assert got[k] == pytest.approx(want[k], rel=1e-14), (alg, args, k)
    # ||G|| = 0 with sigma_L > 0: k_total = 0 (the log's argument clamped to 1), not 0 * log 0
    assert theory_schedule("DFGM", 1e-2, 1.0, 1.0, 40.0, 0.5, 2.0, 0.0)["k_total"] == 0
    # Q = I is Case 1, Q = 0 Case 2, Q = diag(1, 1e-12) Case 2 under tau_pd
    sched = lambda lmin, lmax: theory_schedule("DGM", 1e-2, 1.0, 1.0, 1.0, 0.0, 2.0, 1.0, lmin, lmax)["case_id"]
    assert (sched(1.0, 1.0), sched(0.0, 0.0), sched(1e-12, 1.0)) == (1, 2, 2)
    out = _lib.Schedule()
    assert lib.duquad_theory_schedule(1, -1.0, 1, 1, 1, 0, 1, 1, 0, 0, C.byref(out)) == _lib.DUQUAD_EINVAL
    assert lib.duquad_theory_schedule(1, 1e-2, 1, 1, 1, float("nan"), 1, 1, 0, 0, C.byref(out)) == _lib.DUQUAD_EINVAL
    assert lib.duquad_theory_schedule(7, 1e-2, 1, 1, 1, 0, 1, 1, 0, 0, C.byref(out)) == _lib.DUQUAD_EINVAL
    assert lib.duquad_theory_schedule(1, 1e-2, 1, 1, 1, 0, 1, 1, 0, -1.0, C.byref(out)) == _lib.DUQUAD_EINVAL
    assert lib.duquad_status_string(_lib.DUQUAD_EMAXITER).startswith(b"inner iteration cap")


def test_theory_bounds_host_only(lib):
    """duquad_theory_bounds is host arithmetic: the oracle's theorem1 / drift / feasibility bounds
    (pinned against actual DFOM runs in tests/test_oracle_pins.py)."""
    from oracle import dfom as O
    from paper_1504_05708_b200 import theory_bounds, _lib
    for alg in ("DGM", "DFGM"):
        for k, L_d, R_d, e in [(1, 2.0, 3.0, 1e-3), (17, 0.7, 12.0, 0.0), (400, 1.0, 0.0, 1e-6)]:
            b = theory_bounds(alg, k, L_d, R_d, e)
            assert b["dual_gap"] == pytest.approx(O.theorem1_bound(alg, k, L_d, R_d, e), rel=1e-14)
            assert b["drift"] == pytest.approx(O.drift_bound(k, L_d, R_d, e), rel=1e-14)
            assert b["feas_last"] == pytest.approx(O.feas_last_bound(alg, k, L_d, R_d, e), rel=1e-14, abs=1e-300)
            assert b["feas_avg"] == pytest.approx(O.feas_avg_bound(alg, k, L_d, R_d, e), rel=1e-14, abs=1e-300)
    for bad in [(0, 1.0, 1.0, 0.0), (3, 0.0, 1.0, 0.0), (3, 1.0, -1.0, 0.0), (3, 1.0, 1.0, float("nan"))]:
        with pytest.raises(_lib.DuquadError):
            theory_bounds("DGM", *bad)
