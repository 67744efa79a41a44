"""Seeded synthetic QP generators shared by the CPU oracle and the CUDA path.

This module holds NO arithmetic of the DuQuad method (no projections, no
gradients, no dual updates): it only draws random problem data with the
shapes, value distributions and structure of BASELINE.json's five configs
(recipes pinned in SURVEY.md §8(d) and restated in DESIGN.md §3).  Both the
oracle (`oracle/`) and the product path (`paper_1504_05708_b200/`) consume
the arrays it returns; neither imports the other.

Cone tags follow the paper's K (Eq. original_primal):
0 = ZERO (equality row, K = {0}), 1 = NONPOS (inequality row, K = R_-).

Draw order is part of the contract: changing it changes every fixture.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

ZERO = 0
NONPOS = 1


@dataclass
class DenseQP:
    """min 1/2 u'Qu + q'u, u in [lb, ub], Gu + g in K."""

    Q: np.ndarray            # n x n, symmetric
    q: np.ndarray            # n   (or n x B for a batch sharing Q, G)
    G: np.ndarray            # p x n
    g: np.ndarray            # p   (or p x B)
    lb: np.ndarray           # n
    ub: np.ndarray           # n
    cone: np.ndarray         # p uint8 (ZERO / NONPOS)
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.Q.shape[0]

    @property
    def p(self) -> int:
        return self.G.shape[0]


@dataclass
class SparseQP:
    """CSR variant (config 4).  Arrays are scipy.sparse.csr_matrix."""

    Q: object
    q: np.ndarray
    G: object
    g: np.ndarray
    lb: np.ndarray
    ub: np.ndarray
    cone: np.ndarray
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.Q.shape[0]

    @property
    def p(self) -> int:
        return self.G.shape[0]


def dense_ineq(n: int, p: int, seed: int = 0, shift: float = 0.1,
               box: float = 1.0, name: str = "") -> DenseQP:
    """Configs 0/1 (and 2 on the host): strictly feasible random inequality QP.

    Draws, in order, from numpy.random.default_rng(seed):
      M (n x n) ~ N(0,1); q (n) ~ N(0,1); G (p x n) ~ N(0,1);
      x0 (n) ~ U(-0.5, 0.5); slack (p) ~ U(0.1, 1).
    Then Q = M'M/n + shift*I (symmetrised), g = -G x0 - slack, so x0 is
    strictly feasible (G x0 + g = -slack < 0) and inside the box.
    """
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((n, n))
    q = rng.standard_normal(n)
    G = rng.standard_normal((p, n))
    x0 = rng.uniform(-0.5, 0.5, n)
    slack = rng.uniform(0.1, 1.0, p)
    Q = M.T @ M / n + shift * np.eye(n)
    Q = 0.5 * (Q + Q.T)
    g = -(G @ x0) - slack
    lb = np.full(n, -box)
    ub = np.full(n, box)
    cone = np.full(p, NONPOS, dtype=np.uint8)
    return DenseQP(Q, q, G, g, lb, ub, cone, name=name or f"dense_ineq_n{n}_p{p}_s{seed}",
                   meta=dict(seed=seed, shift=shift, x0=x0))


def dense_ineq_torch(n: int, p: int, seed: int = 0, shift: float = 0.05,
                     box: float = 1.0, device: str = "cuda"):
    """Config 2 at full size, drawn on the device with torch's generator.

    Same recipe as `dense_ineq` (M, q, G ~ N(0,1); x0 ~ U(-.5,.5);
    slack ~ U(.1,1); Q = M'M/n + shift I; g = -G x0 - slack) but drawn with
    torch.Generator(device).manual_seed(seed) because the 16384^3 product
    M'M would take minutes on the host.  Returns a dict of fp64 torch
    tensors on `device`.  The numbers differ from `dense_ineq` with the same
    seed (different generator); both sides of any parity test consume the
    SAME returned tensors (copied to the host for the oracle).
    """
    import torch

    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    f64 = torch.float64
    M = torch.randn((n, n), generator=gen, dtype=f64, device=device)
    q = torch.randn((n,), generator=gen, dtype=f64, device=device)
    G = torch.randn((p, n), generator=gen, dtype=f64, device=device)
    x0 = torch.rand((n,), generator=gen, dtype=f64, device=device) - 0.5
    slack = 0.1 + 0.9 * torch.rand((p,), generator=gen, dtype=f64, device=device)
    Q = torch.mm(M.t(), M)
    del M
    Q.div_(n)
    Q.diagonal().add_(shift)
    Q = 0.5 * (Q + Q.t())
    g = -(G @ x0) - slack
    lb = torch.full((n,), -box, dtype=f64, device=device)
    ub = torch.full((n,), box, dtype=f64, device=device)
    cone = torch.full((p,), NONPOS, dtype=torch.uint8, device=device)
    return dict(Q=Q, q=q, G=G, g=g, lb=lb, ub=ub, cone=cone)


def mpc_batch(B: int, seed: int = 0, nx: int = 12, nu: int = 4, N: int = 30,
              xbound: float = 5.0, ubound: float = 1.0, rweight: float = 0.1):
    """Config 3: B condensed-MPC QPs sharing Q and G (north_star (c)).

    Draws: Ma (nx x nx), Bu (nx x nu) ~ N(0,1); A = 0.95 Ma / specrad(Ma).
    x_k = A^k x0 + sum_{j<k} A^{k-1-j} Bu u_j for k = 1..N, so the stacked
    state is Phi x0 + Gamma u.  Cost sum ||x_k||^2 + rweight ||u||^2 gives
    (after a factor 1/2) Q = Gamma'Gamma + rweight I, q_b = Gamma' Phi x0_b.
    State bounds |x_k| <= xbound give G = [Gamma; -Gamma],
    g_b = [Phi x0_b - xbound; -Phi x0_b - xbound]; box |u| <= ubound.
    Per QP b (in order) x0_b ~ U(-3,3)^nx, redrawn while
    ||Phi x0_b||_inf > 0.9 xbound, so u = 0 is strictly feasible.
    Returns a DenseQP whose q is n x B and g is p x B (column b = QP b).
    """
    rng = np.random.default_rng(seed)
    Ma = rng.standard_normal((nx, nx))
    Bu = rng.standard_normal((nx, nu))
    A = 0.95 * Ma / np.max(np.abs(np.linalg.eigvals(Ma)))
    n = nu * N
    Apow = [np.eye(nx)]
    for _ in range(N):
        Apow.append(A @ Apow[-1])
    Gamma = np.zeros((nx * N, n))
    Phi = np.zeros((nx * N, nx))
    for k in range(1, N + 1):
        Phi[(k - 1) * nx:k * nx, :] = Apow[k]
        for j in range(k):
            Gamma[(k - 1) * nx:k * nx, j * nu:(j + 1) * nu] = Apow[k - 1 - j] @ Bu
    Q = Gamma.T @ Gamma + rweight * np.eye(n)
    Q = 0.5 * (Q + Q.T)
    G = np.vstack([Gamma, -Gamma])
    X0 = np.zeros((nx, B))
    for b in range(B):
        while True:
            x0 = rng.uniform(-3.0, 3.0, nx)
            if np.max(np.abs(Phi @ x0)) <= 0.9 * xbound:
                break
        X0[:, b] = x0
    PX = Phi @ X0
    q = Gamma.T @ PX
    g = np.vstack([PX - xbound, -PX - xbound])
    lb = np.full(n, -ubound)
    ub = np.full(n, ubound)
    cone = np.full(2 * nx * N, NONPOS, dtype=np.uint8)
    return DenseQP(Q, q, G, g, lb, ub, cone, name=f"mpc_B{B}_s{seed}",
                   meta=dict(seed=seed, A=A, Bu=Bu, X0=X0, nx=nx, nu=nu, N=N))


def sparse_banded_eq(n: int = 1_000_000, p: int = 500_000, seed: int = 0,
                     half_band: int = 5, nnz_per_row: int = 8, box: float = 1.0) -> SparseQP:
    """Config 4: banded symmetric Q (2*half_band+1 nnz/row), random sparse G, K = {0}.

    Draws, in order: diag (n) ~ U(0, 0.5) (+1.5); for d = 1..half_band an
    upper band (n-d) ~ U(-0.1, 0.1), mirrored below; G column indices
    (p x nnz_per_row) ~ integers[0, n), duplicates within a row redrawn row by
    row in row order, then sorted; G values (p x nnz_per_row) ~ N(0,1);
    x0 (n) ~ U(-0.5, 0.5); q (n) ~ N(0,1).  g = -G x0 (x0 feasible).
    Gershgorin: lambda(Q) in [1.5 - 10*0.1, 2 + 10*0.1] = [0.5, 3].
    """
    import scipy.sparse as sp

    rng = np.random.default_rng(seed)
    diag = 1.5 + rng.uniform(0.0, 0.5, n)
    bands = [rng.uniform(-0.1, 0.1, n - d) for d in range(1, half_band + 1)]
    offsets = [0] + [d for d in range(1, half_band + 1)] + [-d for d in range(1, half_band + 1)]
    data = [diag] + bands + bands
    Q = sp.diags(data, offsets, shape=(n, n), format="csr")
    Q.sort_indices()
    cols = rng.integers(0, n, size=(p, nnz_per_row))
    srt = np.sort(cols, axis=1)
    dup_rows = np.nonzero((srt[:, 1:] == srt[:, :-1]).any(axis=1))[0]
    for i in dup_rows:
        while len(np.unique(cols[i])) < nnz_per_row:
            cols[i] = rng.integers(0, n, size=nnz_per_row)
    cols = np.sort(cols, axis=1)
    vals = rng.standard_normal((p, nnz_per_row))
    indptr = np.arange(0, p * nnz_per_row + 1, nnz_per_row, dtype=np.int64)
    G = sp.csr_matrix((vals.ravel(), cols.ravel(), indptr), shape=(p, n))
    x0 = rng.uniform(-0.5, 0.5, n)
    q = rng.standard_normal(n)
    g = -(G @ x0)
    lb = np.full(n, -box)
    ub = np.full(n, box)
    cone = np.full(p, ZERO, dtype=np.uint8)
    return SparseQP(Q, q, G, g, lb, ub, cone, name=f"sparse_banded_n{n}_p{p}_s{seed}",
                    meta=dict(seed=seed, x0=x0))


def tiny(n: int, p: int, seed: int, kind: str = "ineq", box: float = 1.0,
         shift: float = 0.1, psd_rank: Optional[int] = None) -> DenseQP:
    """Small random QPs for oracle pins and edge cases.

    kind: 'ineq' (all NONPOS rows, strictly feasible), 'eq' (all ZERO rows,
    x0 feasible), 'mixed' (alternating ZERO/NONPOS).  psd_rank < n gives a
    singular Q (Case 2 of PAPER.md:257-259; needs rho > 0).
    Draws: M (r x n), q (n), G (p x n) ~ N(0,1); x0 ~ box*U(-.5,.5)^n (inside U);
    slack ~ U(.1,1)^p.
    """
    rng = np.random.default_rng(seed)
    r = n if psd_rank is None else psd_rank
    M = rng.standard_normal((r, n))
    q = rng.standard_normal(n)
    G = rng.standard_normal((p, n))
    x0 = box * rng.uniform(-0.5, 0.5, n)
    slack = rng.uniform(0.1, 1.0, p)
    Q = M.T @ M / n + (shift if psd_rank is None else 0.0) * np.eye(n)
    Q = 0.5 * (Q + Q.T)
    if kind == "ineq":
        cone = np.full(p, NONPOS, dtype=np.uint8)
    elif kind == "eq":
        cone = np.full(p, ZERO, dtype=np.uint8)
    elif kind == "mixed":
        cone = np.array([ZERO if i % 2 == 0 else NONPOS for i in range(p)], dtype=np.uint8)
    else:
        raise ValueError(kind)
    g = -(G @ x0) - np.where(cone == NONPOS, slack, 0.0)
    lb = np.full(n, -box)
    ub = np.full(n, box)
    return DenseQP(Q, q, G, g, lb, ub, cone, name=f"tiny_{kind}_n{n}_p{p}_s{seed}",
                   meta=dict(seed=seed, x0=x0))


# Named configs of BASELINE.json (index = position in BASELINE.json "configs").
CONFIGS = {
    0: dict(n=50, p=25, shift=0.1, alg="DFGM", rho=1.0, outer=200, inner=50, lambda_min_lb=0.1),
    1: dict(n=2000, p=1000, shift=0.1, alg="DFGM", rho=1.0, outer=400, inner=50, lambda_min_lb=0.1),
    2: dict(n=16384, p=8192, shift=0.05, alg="DFGM", rho=1.0, outer=100, inner=100, lambda_min_lb=0.05),
    3: dict(B=8192, alg="DFGM", rho=1.0, outer=50, inner=20, lambda_min_lb=0.1),
    4: dict(n=1_000_000, p=500_000, alg="DFGM", rho=5.0, outer=300, inner=50, lambda_min_lb=0.5),
}
