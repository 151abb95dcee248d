"""Level-space diagnostics of the quantised state -- TEST INFRASTRUCTURE ONLY
(only tests/, __graft_entry__.smoke() and bench.py may import anything under
oracle/).  Plain numpy, float64, written in the order of PAPER.md's
Supplementary Information "Entropy and Statistical Structure":

    p_k = #{i | q_i = k} / N                                  (Eq. pk_definition)
    S = -sum_k p_k log p_k                                     (Eq. discrete_entropy)
    N_eff = exp(S)                                             (Eq. neff)
    N_{k'k} = #{i | q^n_i = k and q^{n+1}_i = k'}              (Def. level_transition)
    M_{k'k} = N_{k'k} / c^n_k  (0 when c^n_k = 0)              (Eq. empirical_M)
    rho = max_{k'} |sum_k M_{k'k} - 1|                          (Rem. doubly_stochastic)
    dS/dt = (S^{n+1} - S^n) / dt                                (Eq. entropy_rate)

Reading A17: the max in rho runs over the union of the supports of
p^n and p^{n+1} -- the finite state space Thm. S2's proof restricts M^n to
(P:770); every level outside both supports has an all-zero row and column and
would contribute the constant |0 - 1| = 1 to an unrestricted max.
Pins: tests/test_oracle_diagnostics.py (Prop. S1(i) closed form, scipy's
entropy, the column-stochastic / p^{n+1} = M p^n identities of Def. S2 on
non-symmetric data, brute-force pair counting, Thm. S2 on constructed doubly
stochastic mixing)."""
from __future__ import annotations

import numpy as np


def level_counts(q) -> tuple[np.ndarray, np.ndarray]:
    """(levels k, counts c_k) over the occupied levels, ascending k."""
    q = np.asarray(q).ravel()
    return np.unique(q, return_counts=True)


def level_distribution(q) -> tuple[np.ndarray, np.ndarray]:
    """(levels k, p_k = c_k / N) -- Eq. pk_definition."""
    k, c = level_counts(q)
    return k, c.astype(np.float64) / float(np.asarray(q).size)


def entropy(q) -> float:
    """S = -sum_k p_k log p_k -- Eq. discrete_entropy (natural log)."""
    _, p = level_distribution(q)
    return float(-np.sum(p * np.log(p)))


def n_eff(q) -> float:
    """N_eff = exp(S) -- Eq. neff."""
    return float(np.exp(entropy(q)))


def transition_counts(q0, q1) -> dict[tuple[int, int], int]:
    """{(k', k): N_{k'k}} over the non-zero entries -- Def. level_transition."""
    q0 = np.asarray(q0).ravel()
    q1 = np.asarray(q1).ravel()
    assert q0.shape == q1.shape
    pairs, cnt = np.unique(np.stack([q1, q0], axis=1), axis=0, return_counts=True)
    return {(int(a), int(b)): int(c) for (a, b), c in zip(pairs, cnt)}


def transition_matrix(q0, q1) -> tuple[np.ndarray, np.ndarray]:
    """(levels, M) with M[i, j] = M_{levels[i], levels[j]} on the union of the
    two supports -- Eq. empirical_M (M_{k'k} = 0 where c^n_k = 0)."""
    k0, c0 = level_counts(q0)
    k1, _ = level_counts(q1)
    levels = np.union1d(k0, k1)
    index = {int(k): i for i, k in enumerate(levels)}
    c = dict(zip(k0.tolist(), c0.tolist()))
    M = np.zeros((levels.size, levels.size))
    for (kp, k), nkk in transition_counts(q0, q1).items():
        M[index[kp], index[k]] = nkk / c[k]
    return levels, M


def row_sum_defect(q0, q1) -> float:
    """rho = max_{k'} |sum_k M_{k'k} - 1| over the union of the supports (A17)."""
    _, M = transition_matrix(q0, q1)
    return float(np.max(np.abs(M.sum(axis=1) - 1.0)))


def entropy_rate(q0, q1, dt: float) -> float:
    """(S^{n+1} - S^n) / dt -- Eq. entropy_rate."""
    return (entropy(q1) - entropy(q0)) / dt
