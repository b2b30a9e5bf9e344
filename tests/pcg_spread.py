"""Test helper: the oracle PCG's own iteration-count spread under reorderings of the unknowns (DESIGN.md
reading R15).  Calls only oracle/ code."""
import numpy as np

from oracle import solvers


def oracle_iteration_spread(A, b, tol, maxit, precond, lam, ref, m, seeds=(1, 2, 3, 4, 5), true_res=None):
    """Oracle PCG iteration counts on the system as given and under random symmetric permutations of the
    unknowns (P A P^T, P b): the same mathematics with every sum in a different order.  Returns (x of the
    unpermuted solve, its stats, the sorted list of counts).  With a list `true_res`, appends the true
    relative residual ||b - A x|| / ||b|| of every sample (the rounding drift of the recursive residual)."""
    n = b.size
    dinv = 1.0 / A.diagonal() if precond == 1 else None
    Pb = solvers.inverse_mass_preconditioner(m["VX"], m["VY"], m["EToV"], ref, lam) if precond == 2 else None
    x, st = solvers.pcg(lambda v: A @ v, b, tol, maxit, dinv=dinv, apply_P=Pb)
    counts = [st["iterations"]]
    nb = np.linalg.norm(b)
    if true_res is not None:
        true_res.append(np.linalg.norm(b - A @ x) / nb)
    for seed in seeds:
        perm = np.random.default_rng(seed).permutation(n)
        inv = np.empty_like(perm)
        inv[perm] = np.arange(n)
        Ap = A[perm][:, perm].tocsr()
        if precond == 2:
            def P(r, perm=perm, inv=inv):
                return Pb(r[inv])[perm]
        else:
            P = None
        xp, sp = solvers.pcg(lambda v: Ap @ v, b[perm], tol, maxit, dinv=None if dinv is None else dinv[perm], apply_P=P)
        counts.append(sp["iterations"])
        if true_res is not None:
            true_res.append(np.linalg.norm(b[perm] - Ap @ xp) / nb)
    return x, st, sorted(counts)


def check_iterations(gpu_it, it_o, counts):
    """North star: +-1 of the oracle.  Where the oracle itself moves under a reordering of the unknowns, the
    GPU count is one more rounding-order realisation of the same CG: it must lie within the oracle's
    sampled range widened by the range's own width w (a handful of samples underestimates the full range;
    w >= 1), i.e. [min - w, max + w] (R15).  Reorder-stable oracle: +-1 exactly."""
    w = max(1, max(counts) - min(counts))
    lo, hi = min(counts) - w, max(counts) + w
    assert lo <= gpu_it <= hi, (gpu_it, it_o, counts)
    if counts[0] == counts[-1]:
        assert abs(gpu_it - it_o) <= 1, (gpu_it, it_o, counts)
