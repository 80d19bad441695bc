"""Figure 2 protocol (SPEC error_curve S:393-401): for the nine
constructed pairs with J = 0.1..0.9 (datagen.fig2_pairs), mean over 200 seeds of
|J-hat_k - J| for k = 1..50, J-hat_k from the first k hashes (slot-prefix reuse,
S:420), against the exact law of an unbiased estimator with P(h_x = h_y) = J
(Theorem 1, Eq. 14-15): J-hat_k ~ Binomial(k, J) / k."""
import math

import numpy as np

K_MAX, REPS = 50, 200


def exact_mae(J: float, k: int) -> float:
    return sum(math.comb(k, m) * J ** m * (1 - J) ** (k - m) * abs(m / k - J) for m in range(k + 1))


def error_curves(sig_of_seed, J):
    """sig_of_seed(seed) -> uint32 [18, K_MAX] signatures of rows x_0..x_8, y_0..y_8.
    Returns (mae [9, K_MAX], z [9, K_MAX]) with z the deviation from the exact
    binomial MAE in standard errors of a 200-seed mean."""
    hits = np.zeros((REPS, 9, K_MAX), np.float64)
    for r in range(REPS):
        s = sig_of_seed(r + 1)
        hits[r] = (s[:9] == s[9:]).astype(np.float64)
    ks = np.arange(1, K_MAX + 1)
    jhat = np.cumsum(hits, axis=2) / ks                    # prefix estimates
    mae = np.abs(jhat - np.asarray(J)[None, :, None]).mean(axis=0)
    z = np.zeros_like(mae)
    for p, Jp in enumerate(J):
        for k in ks:
            e = exact_mae(Jp, int(k))
            var = max(Jp * (1 - Jp) / k - e * e, 1e-12)
            z[p, k - 1] = (mae[p, k - 1] - e) / math.sqrt(var / REPS)
    return mae, z
