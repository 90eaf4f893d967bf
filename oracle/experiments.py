"""Accuracy experiments of Section 4 (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

mse:        Eq. (20): MSE = 1/(3|Omega|) sum_k sum_i (B_k(i) - S_k(i))^2
            (here 1/(d|Omega|) for d channels); "on a logarithmic scale 10 log10(MSE) dB"
            (reading R13).
mse_curve:  the error-vs-T experiment of Fig. 5: for each Monte Carlo
            realisation (a seed of the reading-R9 generator) and each number of trials T_j,
            the MSE between a reference B and Algorithm 1 run with the first T_j draws.
"""
import numpy as np

from . import draws, native


def mse(B, S):
    """Eq. (20) over all channels and pixels (fp64)."""
    B = np.asarray(B, dtype=np.float64)
    S = np.asarray(S, dtype=np.float64)
    return float(np.mean((B - S) ** 2))


def mse_curve(f, ref, Q, alpha, N, seeds, t_list, sigma_s, spatial="gaussian", sampler="iid", M=None):
    """(len(seeds), len(t_list)) MSEs; realisation r draws M (default max T) samples with
    seeds[r] (iid: reading R9, stratified over the M strata: reading R17) and checkpoint j uses
    the first t_list[j] of them (Alg. 1 run afresh on each prefix)."""
    d = f.shape[0]
    M = int(max(t_list)) if M is None else int(M)
    out = np.empty((len(seeds), len(t_list)))
    for r, s in enumerate(seeds):
        Y = (draws.y_draws if sampler == "iid" else draws.stratified_y_draws)(int(s), M, d, N)
        for j, T in enumerate(t_list):
            S, _, _ = native.mcsf_full(f, Q, alpha, N, Y[:T], sigma_s, spatial=spatial)
            out[r, j] = mse(ref, S)
    return out
