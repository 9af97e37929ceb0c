"""Prototype 2: heavy pole explicit, scalar solve of the 3-pole model by
safeguarded Newton on G(x) = F(x) (pa - x)(pb - x)."""
import sys
import numpy as np
from secular_port import root as root_old

EPS = np.finfo(np.float64).eps
NEWTON = 0
CALLS = 0


def solve3(c, pa, sa, pb, sb, ph, sh, L, U, x0, nmax=8):
    """root in (L, U) of c + sa/(pa-x) + sb/(pb-x) + sh/(ph-x); pa <= L < U <= pb; ph outside [pa, pb].
    Returns (x, inner iterations) or (None, n)."""
    global NEWTON
    def G(x):
        rh = 1.0 / (ph - x)
        B = c + sh * rh
        a = pa - x; b = pb - x
        g = B * a * b + sa * b + sb * a
        dg = sh * rh * rh * a * b - B * (a + b) - sa - sb
        return g, dg
    lo, hi = L, U
    x = x0 if L <= x0 <= U else 0.5 * (L + U)
    global CALLS
    CALLS += 1
    for it in range(nmax):
        g, dg = G(x)
        NEWTON += 1
        if g > 0:
            lo = max(lo, x)
        elif g < 0:
            hi = min(hi, x)
        else:
            return x, it
        if dg != 0:
            xn = x - g / dg
        else:
            xn = 0.5 * (lo + hi)
        if not (lo < xn < hi):
            xn = 0.5 * (lo + hi)
        if abs(xn - x) <= 1e-8 * max(abs(xn), abs(x)):
            return xn, it + 1
        x = xn
    return x, nmax


def quad_lo(ce, sa, sb, de):
    A = ce * de + sa + sb; B = sa * de
    sq = np.sqrt(abs(A * A - 4.0 * B * ce))
    return 2.0 * B / (A + sq) if A > 0 else (A - sq) / (2.0 * ce)


def quad_hi(ce, sa, sb, de):
    A = ce * de - sa - sb; B = sb * de
    sq = np.sqrt(abs(A * A + 4.0 * B * ce))
    return 2.0 * B / (A - sq) if A < 0 else -(A + sq) / (2.0 * ce)


def root(kd, kz2, K, rho, sumz2, j, h, trace=False):
    idx = np.arange(K)
    last = j == K - 1
    if not last:
        de = kd[j + 1] - kd[j]; mid = 0.5 * de
        terms = kz2 / ((kd - kd[j]) - mid)
        s = np.sum(terms)
        if 1.0 + rho * s >= 0.0:
            o, lo, hi = j, 0.0, mid
        else:
            o, lo, hi = j + 1, -mid, 0.0
        dorg = kd[o]
        tau = 0.5 * (lo + hi)
        C = 1.0 / rho + s + kz2[j] / mid - kz2[j + 1] / mid
        heavy = h >= 0 and h != j and h != j + 1
        pa = kd[j] - dorg; pb = kd[j + 1] - dorg
        if heavy:
            C -= terms[h]
            ph = kd[h] - dorg
            ce = C + kz2[h] / (ph - tau)
        else:
            ce = C
        g = quad_lo(ce, kz2[j], kz2[j + 1], de) if o == j else quad_hi(ce, kz2[j], kz2[j + 1], de)
        use3 = False
        if heavy:
            # the heavy pole's own moved eigenvalue (background zero) lies in this interval
            use3 = (C + kz2[h] / (ph - pa)) * (C + kz2[h] / (ph - pb)) < 0
            if use3:
                g, _ = solve3(C, pa, kz2[j], pb, kz2[j + 1], ph, kz2[h], max(lo, pa), min(hi, pb), g)
        if g is not None and lo < g < hi:
            tau = g
    else:
        o, lo, hi = j, 0.0, rho * sumz2 * (1.0 + 4.0 * EPS)
        use3 = False
        dorg = kd[o]
        tau = 0.5 * (lo + hi)
        heavy = False
        msk = np.ones(K, bool); msk[K - 2:] = False
        if heavy:
            msk[h] = False
        sm = np.sum(kz2[msk] / (kd[msk] - kd[K - 1]))
        C = 1.0 / rho + sm; dl = kd[K - 2] - kd[K - 1]; a = kz2[K - 2]; b = kz2[K - 1]
        # poles: pa = dl (<0) weight a, pb = 0 weight b; root x > 0; heavy ph < 0
        if heavy:
            ph = kd[h] - dorg
            # F(x) = C + a/(dl - x) + b/(0 - x) + sh/(ph - x), x in (0, hi): all poles left of x
            def F(x):
                return C + a / (dl - x) + b / (-x) + kz2[h] / (ph - x)
            def dF(x):
                return a / (dl - x) ** 2 + b / x ** 2 + kz2[h] / (ph - x) ** 2
            # Newton on 1/(1 - F/ C)... keep simple: bracketed Newton on x*F(x)
            l2, h2 = 0.0, hi
            x = None
            # start: two-pole guess with heavy frozen at 0
            ce = C + kz2[h] / ph
            if ce > 0:
                Bm = ce * dl + a + b
                sq = np.sqrt(max(Bm * Bm - 4.0 * ce * b * dl, 0.0))
                x = (Bm + sq) / (2.0 * ce) if Bm > 0 else (2.0 * b * dl) / (Bm - sq)
            if x is None or not (l2 < x < h2):
                x = 0.5 * hi
            for _ in range(8):
                fx = F(x)
                if fx < 0: l2 = max(l2, x)
                else: h2 = min(h2, x)
                # Newton on x*F (removes the pole at 0)
                gx = x * fx; dgx = fx + x * dF(x)
                xn = x - gx / dgx if dgx != 0 else 0.5 * (l2 + h2)
                if not (l2 < xn < h2): xn = 0.5 * (l2 + h2)
                if abs(xn - x) <= 4 * EPS * abs(xn):
                    x = xn; break
                x = xn
            if lo < x < hi: tau = x
        elif K >= 2 and C > 0:
            Bm = C * dl + a + b
            sq = np.sqrt(max(Bm * Bm - 4.0 * C * b * dl, 0.0))
            g = (Bm + sq) / (2.0 * C) if Bm > 0 else (2.0 * b * dl) / (Bm - sq)
            if lo < g < hi: tau = g
    it = 0
    heavy_i = (not last) and use3
    while it < 120:
        rdel = 1.0 / ((kd - dorg) - tau)
        t = kz2 * rdel; dt = t * rdel
        psi = rho * np.sum(t[idx <= j]); phi = rho * np.sum(t[idx > j])
        dpsi = rho * np.sum(dt[idx <= j]); dphi = rho * np.sum(dt[idx > j])
        aerr = phi - psi
        f = 1.0 + psi + phi
        if trace: print("   it", it, "tau", tau, "f", f, "lo", lo, "hi", hi)
        if f < 0: lo = max(lo, tau)
        else: hi = min(hi, tau)
        if abs(f) <= 4.0 * EPS * K * (1.0 + aerr): break
        if heavy_i:
            th = rho * t[h]; dth = rho * dt[h]
            if h <= j: psi -= th; dpsi -= dth
            else: phi -= th; dphi -= dth
            Dh = (kd[h] - dorg) - tau; sh = rho * kz2[h]
        D1 = (kd[j] - dorg) - tau
        ok = False; nt = 0.0
        if not last:
            D2 = (kd[j + 1] - dorg) - tau
            q1 = dpsi * D1 * D1; q2 = dphi * D2 * D2
            c = 1.0 + psi - dpsi * D1 + phi - dphi * D2
            ce = c + (sh / Dh if heavy_i else 0.0)
            Bq = ce * (D1 + D2) + q1 + q2
            Cq = D1 * D2 * f
            disc = Bq * Bq - 4.0 * ce * Cq
            eta = None
            if disc >= 0:
                sq = np.sqrt(disc)
                den = Bq + (sq if Bq >= 0 else -sq)
                if den != 0: eta = 2.0 * Cq / den
            if heavy_i:
                L = max(lo - tau, D1); U = min(hi - tau, D2)
                eta, _ = solve3(c, D1, q1, D2, q2, Dh, sh, L, U, 0.0)
            if eta is not None:
                nt = tau + eta; ok = True
        else:
            Pv = -(psi + phi); dP = dpsi + dphi
            if Pv > 0 and dP > 0:
                if heavy_i:
                    sr = Pv * Pv / dP; Dr = -Pv / dP
                    Bm = Dh + Dr + sh + sr
                    Cm = Dh * Dr + sh * Dr + sr * Dh
                    disc = Bm * Bm - 4.0 * Cm
                    if disc >= 0:
                        sq = np.sqrt(disc)
                        eta = 0.5 * (Bm + sq) if Bm > 0 else 2.0 * Cm / (Bm - sq)
                        nt = tau + eta; ok = True
                else:
                    nt = tau + (Pv * Pv - Pv) / dP; ok = True
        if (not ok) or not (lo < nt < hi):
            pos = hi > 0
            a_ = max(lo if pos else -hi, 4.0 * EPS * max(abs(dorg), 1e-300)); b_ = hi if pos else -lo
            nt = (np.sqrt(a_ * b_) if pos else -np.sqrt(a_ * b_)) if b_ > 1e9 * a_ else 0.5 * (lo + hi)
            if trace: print("     safeguard ->", nt)
        if nt == tau or hi - lo <= 2.0 * EPS * max(abs(lo), abs(hi)):
            tau = nt; break
        tau = nt
        it += 1
    return tau, o, it


if __name__ == "__main__":
    P = np.load(sys.argv[1] if len(sys.argv) > 1 else "../gpurun_out/secular_problems.npy")
    nprob = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    allold, allnew, mxo, mxn, maxdiff = [], [], [], [], 0.0
    for pi in range(min(nprob, len(P))):
        o = P[pi]; K = int(o[0])
        if K == 0: continue
        rho = o[1]; kd = o[8:8 + K].copy(); kz2 = o[268:268 + K].copy()
        h = int(np.argmax(kz2))
        if kz2[h] < 0.5 * o[2]: h = -1
        old = [root_old(kd, kz2, K, rho, o[2], j) for j in range(K)]
        new = [root(kd, kz2, K, rho, o[2], j, h) for j in range(K)]
        io = np.array([r[2] for r in old]); inn = np.array([r[2] for r in new])
        for j in range(K):
            lo_ = kd[old[j][1]] + old[j][0]; ln_ = kd[new[j][1]] + new[j][0]
            rel = abs(old[j][0] - new[j][0]) / max(abs(old[j][0]), 1e-300) if old[j][1] == new[j][1] else abs(lo_ - ln_) / max(abs(lo_), 1e-300)
            maxdiff = max(maxdiff, rel)
        allold.append(io); allnew.append(inn); mxo.append(io.max()); mxn.append(inn.max())
    allold = np.concatenate(allold); allnew = np.concatenate(allnew)
    print("old: mean its %.3f, max-per-problem mean %.2f max %d; hist %s" % (allold.mean(), np.mean(mxo), max(mxo), np.bincount(allold)))
    print("new: mean its %.3f, max-per-problem mean %.2f max %d; hist %s" % (allnew.mean(), np.mean(mxn), max(mxn), np.bincount(allnew)))
    print("max rel diff of tau between schemes: %.2e; inner newton evals per root %.2f" % (maxdiff, NEWTON / len(allnew)))
    print("solve3 calls", CALLS, "evals per call", NEWTON / max(CALLS, 1))
    print("per-problem max (old,new):", list(zip(mxo, mxn))[:40])
