"""Pins for the oracle's batched (ensemble) runner `or_run_scalar_batch`
(oracle/fqnm_oracle.c), the checker of every ensemble parity test (ENS-1, cfg1
replicas).  Ensemble mode is B independent problems (BJ north_star "batched
ensembles"; the update of each is Eqs. update_rule / flux difference),
so the batch must equal, row by row, things fixed outside the batch code:

* the unit-Courant exact shift (np.roll, a library routine);
* a step written here by hand from the literal Fraction maps of oracle/rules.py
  (Eq. flux_table, rounded per reading A1) and the flux-difference form
  (P:86-94), with numpy rolls for the periodic neighbours and ghost copies for
  transmissive walls (reading A12) — no code shared with the C loops;
* per-row exact conservation (Thm P:309-333) and row independence.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import PERIODIC, TRANSMISSIVE, rules
from oracle.rules import BURGERS_EO, BURGERS_LF, LINEAR, RHA

CASES = [  # (kind, delta, dt/dx, param, admissible range)
    (LINEAR, "1e-4", Fraction(1, 2), 1, (-3000, 3000)),
    (LINEAR, "1e-3", Fraction(1, 3), -1, (-3000, 3000)),
    (BURGERS_EO, "1e-5", Fraction(4, 15), 1, (-50000, 150000)),
    (BURGERS_LF, "1e-3", Fraction(1, 2), 1, (-900, 900)),
]


def _literal_maps(kind, delta, lam, param, values):
    """phi+ and phi- of every value, from the Fraction definition (rules.phi)."""
    vals = np.unique(values)
    pp = {int(v): rules.phi(kind, delta, lam, int(v), +1, Fraction(param), RHA) for v in vals}
    pm = {int(v): rules.phi(kind, delta, lam, int(v), -1, Fraction(param), RHA) for v in vals}
    return pp, pm


def _hand_step(q, pp, pm, boundary):
    """q' = q - (F_{i+1/2} - F_{i-1/2}), F_{i+1/2} = phi+(q_i) + phi-(q_{i+1})."""
    p = np.vectorize(pp.__getitem__, otypes=[np.int64])(q)
    m = np.vectorize(pm.__getitem__, otypes=[np.int64])(q)
    if boundary == PERIODIC:
        F = p + np.roll(m, -1)                               # F[i] = F_{i+1/2}
        return q - (F - np.roll(F, 1))
    # transmissive ghosts q_{-1} = q_0, q_N = q_{N-1} (reading A12)
    F = p + np.concatenate([m[1:], m[-1:]])                  # F_{i+1/2}, i = 0..N-1
    Fl = np.concatenate([p[:1] + m[:1], F[:-1]])             # F_{i-1/2}
    return q - (F - Fl)


@pytest.mark.parametrize("kind,delta,lam,param,rng_", CASES)
@pytest.mark.parametrize("boundary", [PERIODIC, TRANSMISSIVE])
def test_batch_equals_hand_written_steps(kind, delta, lam, param, rng_, boundary):
    r = oracle.Rule(kind, delta, lam, Fraction(param))
    rng = np.random.default_rng(31)
    B, N, S = 7, 37, 6
    q0 = rng.integers(rng_[0], rng_[1] + 1, (B, N))
    got = r.run(q0, S, boundary)
    want = q0.copy()
    for _ in range(S):
        # maps of every value the trajectory reaches (recomputed each step; small sets)
        pp, pm = _literal_maps(kind, delta, lam, param, want)
        want = np.stack([_hand_step(row, pp, pm, boundary) for row in want])
    assert np.array_equal(got, want)


def test_batch_unit_courant_is_row_wise_roll():
    r = oracle.Rule(LINEAR, "0.01", 1)
    rng = np.random.default_rng(5)
    q = rng.integers(-10**6, 10**6, (9, 64))
    assert np.array_equal(r.run(q, 11), np.roll(q, 11, axis=1))
    assert np.array_equal(r.run(q, 64), q)                  # N periodic steps return the state


@pytest.mark.parametrize("kind,delta,lam,param,rng_", CASES)
def test_batch_rows_are_independent_and_conserve(kind, delta, lam, param, rng_):
    r = oracle.Rule(kind, delta, lam, Fraction(param))
    rng = np.random.default_rng(44)
    B, N, S = 16, 200, 50
    q0 = rng.integers(rng_[0], rng_[1] + 1, (B, N))
    out = r.run(q0, S)
    assert np.array_equal(out.sum(axis=1), q0.sum(axis=1))             # per-row conservation
    q1 = q0.copy()
    q1[3] = rng.integers(rng_[0], rng_[1] + 1, N)                      # perturb one problem
    out1 = r.run(q1, S)
    keep = np.arange(B) != 3
    assert np.array_equal(out1[keep], out[keep])
    # threads do not change the result (one problem per thread, any schedule)
    assert np.array_equal(r.run(q0, S, nthreads=1), out)
    assert np.array_equal(r.run(q0, S, nthreads=3), out)
