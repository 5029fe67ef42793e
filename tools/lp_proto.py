"""numpy mirror of the PDHG iteration in csrc/lp.cu, for tuning the restart /
primal-weight heuristics on the CPU (development tool; not used by the product
or the tests).

usage: python tools/lp_proto.py [seed n k t_max]
"""
import sys

import numpy as np


def pdhg(A, mu_min, p, t_max, eps=1e-8, max_iter=200000, M=64, omega=None, eta=0.999, verbose=False,
         scaled=True, presolve=False):
    n, k = A.shape
    p = np.full(n, p) if np.ndim(p) == 0 else p
    tau = eta / (A.sum(0) + 1.0)
    sig1 = eta / (A.sum(1) + 1.0)
    sig2 = eta / k
    qn = np.sqrt(n * mu_min ** 2 + t_max ** 2)
    # weights of the scaled problem x~ = T^-1/2 x, y~ = S^-1/2 y (PDLP measures in that space)
    wt, ws_, wy, wb = (1 / tau, 1 / eta, 1 / sig1, 1 / sig2) if scaled else (1.0, 1.0, 1.0, 1.0)
    if omega is None:
        cs = np.sqrt((tau * 1.0).sum() + (eta * p ** 2).sum()) if scaled else np.sqrt(k + (p ** 2).sum())
        qs = np.sqrt((sig1 * mu_min ** 2).sum() + sig2 * t_max ** 2) if scaled else qn
        omega = cs / qs if scaled else 1.0
    cn = np.sqrt(k + (p ** 2).sum())
    t = np.zeros(k); s = np.zeros(n); y = np.zeros(n); yb = 0.0
    if presolve:  # rows no vantage sees: σ_i = μ_min, y_i = p_i are optimal and fixed points
        z = A.sum(1) == 0
        s[z] = mu_min
        y[z] = p[z]
    mu = A @ t; S = t.sum()
    gT = A.T @ y
    avg = None
    m = 0
    t_last, s_last, y_last, yb_last = t.copy(), s.copy(), y.copy(), yb
    hist = []

    def score(t_, s_, y_, yb_, mu_, S_, gT_):
        rp = np.sqrt((np.maximum(0, mu_min - mu_ - s_) ** 2).sum() + max(0, S_ - t_max) ** 2)
        rd = np.sqrt((np.maximum(0, y_ - p) ** 2).sum() + (np.maximum(0, gT_ - yb_ - 1) ** 2).sum())
        po = S_ + p @ s_
        do = mu_min * y_.sum() - t_max * yb_
        gap = abs(po - do)
        rel = (rp / (1 + qn), rd / (1 + cn), gap / (1 + abs(po) + abs(do)))
        return np.sqrt(omega * rp ** 2 + rd ** 2 / omega + gap ** 2), rel, po

    kkt_restart = score(t, s, y, yb, mu, S, gT)[0]
    prev = np.inf
    it = it_r = 0
    restarts = 0
    while it < max_iter:
        for _ in range(M):
            w = 1.0 / (m + 1)
            tn = np.maximum(0, t - tau / omega * (1 - gT + yb))
            if avg is None:
                avg = [tn.copy(), gT.copy(), s.copy(), mu.copy(), y.copy(), yb, S]
            avg[0] += w * (tn - avg[0]); avg[1] += w * (gT - avg[1]); avg[5] += w * (yb - avg[5])
            t = tn
            Sn = t.sum()
            mun = A @ t
            sn = np.maximum(0, s - eta / omega * (p - y))
            kxo = mu + s; kxn = mun + sn
            yn = np.maximum(0, y + omega * sig1 * (mu_min - 2 * kxn + kxo))
            avg[2] += w * (sn - avg[2]); avg[3] += w * (mun - avg[3]); avg[4] += w * (y - avg[4])
            ybn = max(0.0, yb + omega * sig2 * (2 * Sn - S - t_max))
            avg[6] += w * (Sn - avg[6])
            mu, s, y, S, yb = mun, sn, yn, Sn, ybn
            m += 1
            gT = A.T @ y
        it += M
        kc, relc, poc = score(t, s, y, yb, mu, S, gT)
        ka, rela, poa = score(avg[0], avg[2], avg[4], avg[5], avg[3], avg[6], avg[1])
        hist.append((it, max(relc), max(rela)))
        if verbose and it % (M * 50) == 0:
            print(it, f"omega={omega:.3g}", "cur", ["%.2e" % x for x in relc], "avg", ["%.2e" % x for x in rela],
                  poc, poa)
        if max(relc) <= eps:
            return dict(t=t, obj=poc, it=it, restarts=restarts, omega=omega, hist=hist)
        if max(rela) <= eps:
            return dict(t=avg[0], obj=poa, it=it, restarts=restarts, omega=omega, hist=hist)
        avg_better = ka < kc
        cand = min(ka, kc)
        do = cand <= 0.2 * kkt_restart or (cand <= 0.8 * kkt_restart and cand > prev) or (it - it_r) >= 0.36 * it
        prev = cand
        if do:
            if avg_better:
                t, gT_, s, mu, y, yb, S = (avg[0].copy(), None, avg[2].copy(), avg[3].copy(), avg[4].copy(), avg[5],
                                           avg[6])
                gT = A.T @ y
            dx = np.sqrt((wt * (t - t_last) ** 2).sum() + (ws_ * (s - s_last) ** 2).sum())
            dy = np.sqrt((wy * (y - y_last) ** 2).sum() + wb * (yb - yb_last) ** 2)
            if dx > 1e-10 and dy > 1e-10:
                omega = np.exp(0.5 * np.log(dy / dx) + 0.5 * np.log(omega))
            t_last, s_last, y_last, yb_last = t.copy(), s.copy(), y.copy(), yb
            kkt_restart = cand
            prev = np.inf
            it_r = it
            m = 0
            avg = None
            restarts += 1
    return dict(t=t, obj=None, it=it, restarts=restarts, omega=omega, hist=hist)


if __name__ == "__main__":
    seed, n, k, t_max = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])) \
        if len(sys.argv) > 4 else (3, 500, 64, 300.0)
    rng = np.random.default_rng(seed)
    A = (rng.uniform(0.0, 8.0, (n, k)) * (rng.uniform(size=(n, k)) < 0.3)).astype(np.float32).astype(np.float64)
    A[np.arange(n), rng.integers(0, k, n)] += rng.uniform(0.5, 2.0, n)
    p = 10.0 * float(np.linalg.norm(A))
    sys.path.insert(0, ".")
    from oracle import lp as OLP
    ref = OLP.solve(A, 280.0, p, t_max)
    print("ref obj", ref["obj"], "y_b", ref["y_budget"])
    r = pdhg(A, 280.0, p, t_max, verbose=True, max_iter=int(sys.argv[5]) if len(sys.argv) > 5 else 50000)
    print(r["it"], r["restarts"], r["obj"], r["omega"])


def c3_matrix(seed):
    """(N, K) oracle A of a C3 world (2D oracle)."""
    sys.path.insert(0, ".")
    from oracle import oracle as O
    from synth import configs
    c = configs.c3(seed)
    pat = O.extruded_patches(c["scene"])
    v = O.vantage(c["scene"], c["vantage"])
    return O.irradiance_matrix(pat, v["samples"][v["feasible"]], mode="2d")["A"]
