"""Oracle-side reference helpers for the parity tests (calls only oracle/)."""
from __future__ import annotations

import numpy as np

import oracle as O


def phi_tab(w) -> np.ndarray:
    return O.phi_table(w.phi, w.N)


def index_fn(w):
    if w.family == "poly":
        return lambda rows: O.polylattice_index_matrix(w.D, w.p, w.z, rows)
    return lambda rows: O.lattice_index_matrix(w.N, w.z, rows)


def X_rows(w, rows, cols=None, tab=None) -> np.ndarray:
    tab = phi_tab(w) if tab is None else tab
    return O.oracle_X_rows(tab, index_fn(w)(np.asarray(rows)), w.A, cols)


def X_full(w, cols=None, tab=None, block=4096) -> np.ndarray:
    tab = phi_tab(w) if tab is None else tab
    return O.oracle_X_full(index_fn(w), tab, w.N, w.A, cols, block=block)


def col_tolerance(w, tab=None, cols=None) -> np.ndarray:
    """north_star: |X_gpu - X_oracle| <= 1e-11 · ||a||_1 · max|φ| per column."""
    tab = phi_tab(w) if tab is None else tab
    A = w.A if cols is None else w.A[:, cols]
    return 1e-11 * np.abs(A).sum(axis=0) * np.abs(tab).max()


def sample_rows(N: int, k: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    extra = rng.choice(N, size=min(k, N), replace=False)
    return np.unique(np.concatenate([[0, 1, 2, N - 1], extra]).astype(np.int64) % N)
