"""CPU: the multi-GPU ZJA search as a resumable state machine (csrc/zja.cu
zja_search_step_kernel: phases m0 -> test 1 -> bisection -> 16-point scan -> fallback
bisection) restated step for step, against the direct search distributed.zja_search
(schedule.cpp:233-263) on monotone and non-monotone discrepancy curves: the same beta,
the same warning, the same number of probes; and the host's batch size for the first
poll (distributed._bisect_probes) never exceeds what the search needs."""
import math

import numpy as np

from paper_2408_12057_b200 import distributed

M0, TEST1, BISECT, SCAN, FALLBACK, DONE = range(6)


def machine(dhat, beta, delta, tol=1e-10):
    """zja_search_step_kernel's transitions; returns (beta_t, warn, probes incl. m0)."""
    z = dict(phase=M0, b2=-1.0, beta=beta, lo=0.0, hi=0.0, root=0.0, scan_i=0, warn=False, chosen=beta, probes=0)

    def bisect_next():
        if z["hi"] - z["lo"] > tol:
            z["b2"] = 0.5 * (z["lo"] + z["hi"])
            return True
        return False

    def start_scan():
        z.update(root=z["lo"], phase=SCAN, scan_i=1)
        z["b2"] = z["beta"] + (z["root"] - z["beta"]) * float(z["scan_i"]) / 16

    while z["phase"] != DONE:
        z["probes"] += 1
        if z["phase"] == M0:  # the log-weights' lse: not a dhat probe
            z.update(phase=TEST1, b2=1.0)
            continue
        x = z["b2"]
        d = dhat(x)
        if z["phase"] == TEST1:
            if d <= delta:
                z.update(chosen=1.0, phase=DONE)
                continue
            z.update(lo=z["beta"], hi=1.0, phase=BISECT)
            if not bisect_next():
                start_scan()
        elif z["phase"] == BISECT:
            z["lo" if d <= delta else "hi"] = x
            if not bisect_next():
                start_scan()
        elif z["phase"] == SCAN:
            if d > delta * (1.0 + 1e-12):
                z.update(warn=True, lo=z["beta"], hi=x, phase=FALLBACK)
                if not bisect_next():
                    z.update(chosen=z["lo"], phase=DONE)
            else:
                z["scan_i"] += 1
                if z["scan_i"] < 16:
                    z["b2"] = z["beta"] + (z["root"] - z["beta"]) * float(z["scan_i"]) / 16
                else:
                    z.update(chosen=z["root"], phase=DONE)
        elif z["phase"] == FALLBACK:
            z["lo" if d <= delta else "hi"] = x
            if not bisect_next():
                z.update(chosen=z["lo"], phase=DONE)
    return z["chosen"], z["warn"], z["probes"]


def curves():
    g = np.random.default_rng(11)
    for _ in range(40):
        a, p = g.uniform(0.1, 50.0), g.uniform(1.0, 3.0)
        yield "monotone", (lambda b2, beta, a=a, p=p: a * max(b2 - beta, 0.0) ** p)
    for _ in range(20):  # a bump: non-monotone, exercises the scan's fallback bisection
        a, c, w = g.uniform(1.0, 10.0), g.uniform(0.2, 0.8), g.uniform(0.01, 0.1)
        yield "bump", (lambda b2, beta, a=a, c=c, w=w: 0.5 * a * (b2 - beta) ** 2
                       + a * math.exp(-((b2 - beta - c * (1 - beta)) / (w * (1 - beta))) ** 2))


def test_state_machine_equals_direct_search():
    seen_warn = 0
    for kind, f in curves():
        for beta in (0.0, 0.3, 0.9, 1.0 - 1e-9):
            for delta in (1e-3, 0.05, 0.5):
                probes = [0]

                def dhat(b2):
                    probes[0] += 1
                    return f(b2, beta)

                want = distributed.zja_search(dhat, beta, delta)
                n_direct = probes[0]
                got_b, got_w, got_p = machine(lambda b2: f(b2, beta), beta, delta)
                assert (got_b, got_w) == want, (kind, beta, delta)
                assert got_p == n_direct + 1  # + the m0 probe
                seen_warn += got_w
                # the first poll's batch (2 + bisection length + 15) is enough for a
                # monotone search and never more than a monotone search can use
                if not got_w and got_b != 1.0:
                    assert got_p <= 2 + distributed._bisect_probes(beta) + 15 + 1
    assert seen_warn > 0  # the non-monotone fallback was exercised
