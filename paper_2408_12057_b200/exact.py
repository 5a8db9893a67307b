"""Closed-form normalising constants of the configured targets (host scalar math,
the analogue of AnnealedTarget::analytic_log_z, src/target.cpp:85-89).

Config 5 (relaxed Ising, ASMC_TARGET_ISING): with u = A y, A = delta I + K (Adj + 4 I),
    p~(y) = exp(-y'Ay/2) prod_i 2cosh(u_i) = sum_s exp(-y'Ay/2 + s'Ay)
so  Z(1) = int p~ = (2 pi)^{n/2} |A|^{-1/2} sum_s exp(s'As/2)
         = (2 pi)^{n/2} |A|^{-1/2} e^{c n/2} Z_Ising(K),    c = delta + 4K,
and y | s ~ N(s, A^{-1}).  |A| from the torus eigenvalues, Z_Ising from Kaufman's
exact finite-torus formula (pinned against brute-force enumeration in
tests/test_ising.py)."""
import math


def ising_log_z(L, K, M=None):
    """log Z of the 2D Ising model on an M x L torus (M rows, default square),
    H = -K sum_<ij> s_i s_j over the 2 M L nearest-neighbour bonds (Kaufman 1949)."""
    m, n = (L if M is None else M), L
    if K == 0.0:
        return m * n * math.log(2.0)

    def gam(k):
        if k == 0:
            return 2.0 * K + math.log(math.tanh(K))
        return math.acosh(math.cosh(2.0 * K) / math.tanh(2.0 * K) - math.cos(math.pi * k / n))

    terms = []
    for par in (1, 0):
        lc, ls, sgn = 0.0, 0.0, 1
        for r in range(n):
            x = 0.5 * m * gam(2 * r + par)
            lc += math.log(2.0 * math.cosh(x))
            sh = 2.0 * math.sinh(x)
            if sh == 0.0:
                ls = -math.inf
            else:
                ls += math.log(abs(sh))
                sgn *= 1 if sh > 0 else -1
        terms += [(1, lc), (sgn, ls)]
    mx = max(l for _, l in terms)
    tot = sum(s * math.exp(l - mx) for s, l in terms if l > -math.inf)
    return math.log(0.5) + 0.5 * m * n * math.log(2.0 * math.sinh(2.0 * K)) + mx + math.log(tot)


def ising_log_det_a(L, K, delta):
    """log |A|, A = delta I + K (Adj + 4 I) on the L x L torus (circulant eigenvalues)."""
    acc = 0.0
    for k1 in range(L):
        for k2 in range(L):
            acc += math.log(delta + K * (4.0 + 2.0 * math.cos(2 * math.pi * k1 / L)
                                         + 2.0 * math.cos(2 * math.pi * k2 / L)))
    return acc


def ising_relaxed_log_z(L, K, delta):
    """log Z(1) of the relaxed target (eta normalised, so log Z(0) = 0)."""
    n = L * L
    c = delta + 4.0 * K
    return 0.5 * n * math.log(2 * math.pi) - 0.5 * ising_log_det_a(L, K, delta) + 0.5 * c * n \
        + ising_log_z(L, K)


K_CRITICAL = 0.5 * math.log(1.0 + math.sqrt(2.0))  # Onsager: 0.44068679...
