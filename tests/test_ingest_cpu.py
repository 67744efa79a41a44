"""Two-sided constraint ingestion; host only."""
import numpy as np
import pytest

from oracle import dfom as O
from paper_1504_05708_b200.ingest import NONPOS, ZERO, raw_multipliers, two_sided


def test_spec_examples():
    # lb = ub = 0, g = 0 -> one ZERO row with g = 0
    ing = two_sided(np.array([[1.0, 2.0]]), [0.0], [0.0], [0.0])
    assert ing.cone.tolist() == [ZERO] and ing.g.tolist() == [0.0]
    # lb = -inf, ub = 1 -> one NONPOS row with g = -1
    ing = two_sided(np.array([[1.0, 2.0]]), [0.0], [-np.inf], [1.0])
    assert ing.cone.tolist() == [NONPOS] and ing.g.tolist() == [-1.0]
    # lb = -1, ub = 1 -> two NONPOS rows, g = (-1, -1), the second row of G negated
    ing = two_sided(np.array([[1.0, 2.0]]), [0.0], [-1.0], [1.0])
    assert ing.cone.tolist() == [NONPOS, NONPOS] and ing.g.tolist() == [-1.0, -1.0]
    assert np.array_equal(ing.G, np.array([[1.0, 2.0], [-1.0, -2.0]]))
    # both sides infinite: the row disappears
    ing = two_sided(np.array([[1.0, 2.0]]), [0.0], [-np.inf], [np.inf])
    assert ing.G.shape[0] == 0


def test_equivalence_on_sample_points():
    """u satisfies the raw interval constraints iff G u + g lies in K, on random points."""
    rng = np.random.default_rng(0)
    m, n = 9, 4
    Gb = rng.standard_normal((m, n))
    gb = rng.standard_normal(m)
    lb = np.array([-1.0, -np.inf, 0.3, -2.0, 0.0, -np.inf, -0.5, 1.0, -1.0])
    ub = np.array([1.0, 0.5, 0.3, np.inf, 2.0, np.inf, 0.5, 1.0, -0.2])
    ing = two_sided(Gb, gb, lb, ub)
    for _ in range(2000):
        u = rng.uniform(-1.5, 1.5, n)
        v = Gb @ u + gb
        raw_ok = bool(np.all((v >= lb - 1e-12) & (v <= ub + 1e-12)) and np.all(np.abs(v[lb == ub] - lb[lb == ub]) < 1e-9))
        r = ing.G @ u + ing.g
        ok = bool(np.all(np.where(ing.cone == ZERO, np.abs(r) < 1e-9, r <= 1e-12)))
        if np.all(lb < ub):   # without equality rows the two tests are exact mirrors
            assert raw_ok == ok
        elif not ok:
            assert not raw_ok


def test_sparse_input_and_errors():
    import scipy.sparse as sp
    Gb = sp.random(6, 5, density=0.5, random_state=1, format="csr")
    gb, lb, ub = np.zeros(6), np.full(6, -1.0), np.ones(6)
    ing = two_sided(Gb, gb, lb, ub)
    dense = two_sided(Gb.toarray(), gb, lb, ub)
    assert np.allclose(ing.G.toarray(), dense.G) and np.array_equal(ing.cone, dense.cone)
    with pytest.raises(ValueError):
        two_sided(np.eye(2), [0.0, 0.0], [1.0, 0.0], [0.0, 1.0])          # lb > ub
    with pytest.raises(ValueError):
        two_sided(np.eye(2), [np.nan, 0.0], [0.0, 0.0], [1.0, 1.0])
    with pytest.raises(ValueError):
        two_sided(np.eye(2), [0.0], [0.0], [1.0])


def test_solution_through_ingestion_satisfies_the_interval_kkt():
    """DFOM (oracle) on the ingested problem: the primal point satisfies the raw intervals and the
    mapped-back multipliers give raw stationarity Q u + q + G_bar' lam_raw ~ 0 (box inactive)."""
    rng = np.random.default_rng(4)
    n, m = 8, 5
    M = rng.standard_normal((n, n))
    Q = M.T @ M / n + 0.5 * np.eye(n)
    q = rng.standard_normal(n)
    Gb = rng.standard_normal((m, n))
    gb = np.zeros(m)
    lb = np.array([-0.2, -np.inf, 0.1, -0.3, 0.0])
    ub = np.array([0.2, 0.1, 0.1, np.inf, 0.4])
    ing = two_sided(Gb, gb, lb, ub)
    box = np.full(n, 50.0)
    L_in, L_d, _ = O.lipschitz_constants(Q, ing.G, 0.0, 0.5)
    r = O.dfom(Q, q, ing.G, ing.g, -box, box, ing.cone, 0.0, O.DFGM, 600, 60, L_in, L_d)
    v = Gb @ r.x_last + gb
    assert np.all(v >= lb - 1e-4) and np.all(v <= ub + 1e-4) and abs(v[2] - 0.1) < 1e-4
    lam_raw = raw_multipliers(r.lam, ing, m)
    assert np.linalg.norm(Q @ r.x_last + q + Gb.T @ lam_raw) < 1e-4
