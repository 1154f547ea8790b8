"""Shared assertions of the parity tests (test infrastructure).

Every comparison reports two numbers (PAPER.md:372-381 defines the error as a
relative L2 over a target set; a single bad target among 10^5 would hide under
it, so the per-element maximum is checked beside it):

* rel_l2 = ||u - ref||_2 / ||ref||_2                        <= tol
* max_rel = max_i |u_i - ref_i| / rms(ref)                  <= MAX_FACTOR * tol

rms(ref) = ||ref||_2 / sqrt(n), so max_rel <= sqrt(n) * rel_l2 always; the bar
MAX_FACTOR * tol (MAX_FACTOR = 10) says no single target carries an error more
than 10x the typical one allowed.
"""
import numpy as np

import oracle

MAX_FACTOR = 10.0


def max_rel(u, ref) -> float:
    u = np.asarray(u); ref = np.asarray(ref)
    rms = float(np.sqrt(np.mean(np.abs(ref) ** 2)))
    return float(np.max(np.abs(u - ref)) / rms)


def assert_close(u, ref, tol, what=""):
    """rel. L2 <= tol and per-element max (RMS-normalised) <= MAX_FACTOR * tol; returns both."""
    u = np.asarray(u); ref = np.asarray(ref)
    assert u.shape == ref.shape, (u.shape, ref.shape)
    e2 = oracle.rel_l2(u, ref)
    em = max_rel(u, ref)
    assert e2 <= tol and em <= MAX_FACTOR * tol, f"{what} rel_l2={e2:.3e} max_rel={em:.3e} (tol {tol:.1e})"
    return e2, em
