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


def halpern(A, mu_min, p, t_max, eps=1e-8, max_iter=200000, M=64, eta=0.999, rho=1.0, verbose=False,
            restart_to_T=True, presolve=False):
    """Reflected restarted Halpern PDHG (Lu & Yang 2024) on the same
    preconditioned operator; restarts on the fixed-point residual."""
    n, k = A.shape
    p = np.full(n, p) if np.ndim(p) == 0 else p
    tau = eta / (A.sum(0) + 1.0)
    sig1 = eta / (A.sum(1) + 1.0)
    sig2 = eta / k
    qn = np.sqrt(n * mu_min ** 2 + t_max ** 2)
    cn = np.sqrt(k + (p ** 2).sum())
    cs = np.sqrt(tau.sum() + (eta * p ** 2).sum())
    qs = np.sqrt((sig1 * mu_min ** 2).sum() + sig2 * t_max ** 2)
    omega = cs / qs
    t = np.zeros(k); s = np.zeros(n); y = np.zeros(n); yb = 0.0
    if presolve:
        z = A.sum(1) == 0
        s[z] = mu_min; y[z] = p[z]

    def T(t, s, y, yb, mu, gT):
        tT = np.maximum(0, t - tau / omega * (1 - gT + yb))
        sT = np.maximum(0, s - eta / omega * (p - y))
        muT = A @ tT
        ST = tT.sum()
        yT = np.maximum(0, y + omega * sig1 * (mu_min - 2 * (muT + sT) + (mu + s)))
        ybT = max(0.0, yb + omega * sig2 * (2 * ST - t.sum() - t_max))
        return tT, sT, yT, ybT, muT, A.T @ yT

    def res(a, b):
        dx = (((a[0] - b[0]) ** 2) / tau).sum() + (((a[1] - b[1]) ** 2) / eta).sum()
        dy = (((a[2] - b[2]) ** 2) / sig1).sum() + (a[3] - b[3]) ** 2 / sig2
        return np.sqrt(omega * dx + dy / omega)

    def kkt(z):
        t_, s_, y_, yb_, mu_, gT_ = z
        S_ = t_.sum()
        rp = np.sqrt((np.maximum(0, mu_min - mu_ - s_) ** 2).sum() + max(0, S_ - t_max) ** 2)
        rd = np.sqrt((np.maximum(0, y_ - p) ** 2).sum() + (np.maximum(0, gT_ - yb_ - 1) ** 2).sum())
        po = S_ + p @ s_
        do = mu_min * y_.sum() - t_max * yb_
        return (rp / (1 + qn), rd / (1 + cn), abs(po - do) / (1 + abs(po) + abs(do))), po

    z = (t, s, y, yb, A @ t, A.T @ y)
    z0 = z
    zT = T(*z)
    r0 = res(z, zT)
    prev = np.inf
    it = it_r = kk = 0
    restarts = 0
    hist = []
    last_anchor = z
    while it < max_iter:
        for _ in range(M):
            zT = T(*z)
            lam = (kk + 1) / (kk + 2)
            z = tuple(lam * ((1 + rho) * a - rho * b) + (1 - lam) * c for a, b, c in zip(zT, z, z0))
            # projections are implied for t, s, y >= 0 only at T; the Halpern mix of feasible points stays >= 0
            kk += 1
        it += M
        zT = T(*z)
        r = res(z, zT)
        rel, po = kkt(zT)
        hist.append((it, max(rel)))
        if verbose and it % (M * 50) == 0:
            print(it, f"omega={omega:.3g} r={r:.3e}", ["%.2e" % x for x in rel], po)
        if max(rel) <= eps:
            return dict(t=zT[0], obj=po, it=it, restarts=restarts, omega=omega, hist=hist)
        do = r <= 0.2 * r0 or (r <= 0.8 * r0 and r > prev) or (it - it_r) >= 0.36 * it
        prev = r
        if do:
            znew = zT if restart_to_T else z
            dx = np.sqrt((((znew[0] - last_anchor[0]) ** 2) / tau).sum() + (((znew[1] - last_anchor[1]) ** 2) / eta).sum())
            dy = np.sqrt((((znew[2] - last_anchor[2]) ** 2) / sig1).sum() + (znew[3] - last_anchor[3]) ** 2 / sig2)
            if dx > 1e-10 and dy > 1e-10:
                omega = np.exp(0.5 * np.log(dy / dx) + 0.5 * np.log(omega))
            z = z0 = last_anchor = znew
            r0 = res(z, T(*z))
            prev = np.inf
            it_r = it
            kk = 0
            restarts += 1
    return dict(t=z[0], obj=None, it=it, restarts=restarts, omega=omega, hist=hist)


def capped_proj(v, w, cap):
    """argmin Σ (t-v)²/w s.t. t >= 0, Σt <= cap  ->  t = max(0, v - λw), λ >= 0 (bisection)."""
    t = np.maximum(0, v)
    if t.sum() <= cap:
        return t, 0.0
    lo, hi = 0.0, float(np.max(v / w))
    for _ in range(100):
        mid = 0.5 * (lo + hi)
        if np.maximum(0, v - mid * w).sum() > cap:
            lo = mid
        else:
            hi = mid
    return np.maximum(0, v - hi * w), hi


def halpern_proj(A, mu_min, p, t_max, eps=1e-8, max_iter=200000, M=64, eta=0.999, rho=1.0, verbose=False,
                 alg="halpern"):
    """Budget Σt <= T_max enforced by projection in the primal step (no budget dual row)."""
    n, k = A.shape
    p = np.full(n, p) if np.ndim(p) == 0 else p
    tau = eta / (A.sum(0) + 1e-30)
    tau = np.minimum(tau, eta / 1e-6)
    sig1 = eta / (A.sum(1) + 1.0)
    qn = np.sqrt(n * mu_min ** 2 + t_max ** 2)
    cn = np.sqrt(k + (p ** 2).sum())
    cs = np.sqrt(tau.sum() + (eta * p ** 2).sum())
    qs = np.sqrt((sig1 * mu_min ** 2).sum())
    omega = cs / qs
    t = np.zeros(k); s = np.zeros(n); y = np.zeros(n)

    def T(t, s, y, mu, gT):
        tT, lam = capped_proj(t - tau / omega * (1 - gT), tau, t_max)
        sT = np.maximum(0, s - eta / omega * (p - y))
        muT = A @ tT
        yT = np.maximum(0, y + omega * sig1 * (mu_min - 2 * (muT + sT) + (mu + s)))
        return (tT, sT, yT, muT, A.T @ yT), lam * omega

    def res(a, b):
        dx = (((a[0] - b[0]) ** 2) / tau).sum() + (((a[1] - b[1]) ** 2) / eta).sum()
        dy = (((a[2] - b[2]) ** 2) / sig1).sum()
        return np.sqrt(omega * dx + dy / omega)

    def kkt(z, yb):
        t_, s_, y_, mu_, gT_ = z
        S_ = t_.sum()
        rp = np.sqrt((np.maximum(0, mu_min - mu_ - s_) ** 2).sum() + max(0, S_ - t_max) ** 2)
        rd = np.sqrt((np.maximum(0, y_ - p) ** 2).sum() + (np.maximum(0, gT_ - yb - 1) ** 2).sum())
        po = S_ + p @ s_
        do = mu_min * y_.sum() - t_max * yb
        return (rp / (1 + qn), rd / (1 + cn), abs(po - do) / (1 + abs(po) + abs(do))), po

    z = (t, s, y, A @ t, A.T @ y)
    z0 = last = z
    zT, yb = T(*z)
    r0 = res(z, zT)
    prev = np.inf
    it = it_r = kk = 0
    restarts = 0
    hist = []
    while it < max_iter:
        for _ in range(M):
            zT, yb = T(*z)
            if alg == "halpern":
                lam = (kk + 1) / (kk + 2)
                z = tuple(lam * ((1 + rho) * a - rho * b) + (1 - lam) * c for a, b, c in zip(zT, z, z0))
            else:
                z = zT
            kk += 1
        it += M
        zT, yb = T(*z)
        r = res(z, zT)
        # the dual budget multiplier: best y_b for the current y (min over the dual residual+objective is
        # awkward); use the projection's multiplier
        rel, po = kkt(zT, yb)
        rel2, po2 = kkt(zT, max(0.0, float(np.max(zT[4] - 1.0))))  # y_b making every t-column dual feasible
        if max(rel2) < max(rel):
            rel = rel2
        hist.append((it, max(rel), rel))
        if max(rel) <= eps:
            return dict(t=zT[0], obj=po, it=it, restarts=restarts, omega=omega, hist=hist)
        do = r <= 0.2 * r0 or (r <= 0.8 * r0 and r > prev) or (it - it_r) >= 0.36 * it
        prev = r
        if do and alg == "halpern":
            znew = zT
            dx = np.sqrt((((znew[0] - last[0]) ** 2) / tau).sum() + (((znew[1] - last[1]) ** 2) / eta).sum())
            dy = np.sqrt((((znew[2] - last[2]) ** 2) / sig1).sum())
            if dx > 1e-10 and dy > 1e-10:
                omega = np.exp(0.5 * np.log(dy / dx) + 0.5 * np.log(omega))
            z = z0 = last = znew
            r0 = res(z, T(*z)[0])
            prev = np.inf
            it_r = it
            kk = 0
            restarts += 1
    return dict(t=z[0], obj=None, it=it, restarts=restarts, omega=omega, hist=hist)
