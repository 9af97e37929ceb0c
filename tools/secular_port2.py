"""Prototype: secular root finder with the heavy pole (argmax z^2) explicit in
the rational model (initial guess and iteration); compared with the device
scheme on dumped problems."""
import sys
import numpy as np
from secular_port import root as root_old

EPS = np.finfo(np.float64).eps


def quad_origin_lo(ce, sa, sb, de):   # poles at 0 (sa) and de (sb); root in (0, de)
    A = ce * de + sa + sb; B = sa * de
    sq = np.sqrt(abs(A * A - 4.0 * B * ce))
    return 2.0 * B / (A + sq) if A > 0 else (A - sq) / (2.0 * ce)


def quad_origin_hi(ce, sa, sb, de):   # poles at -de (sa) and 0 (sb); root in (-de, 0)
    A = ce * de - sa - sb; B = sb * de
    sq = np.sqrt(abs(A * A + 4.0 * B * ce))
    return 2.0 * B / (A - sq) if A < 0 else -(A + sq) / (2.0 * ce)


def root(kd, kz2, K, rho, sumz2, j, h, nfix=3, trace=False):
    """h: heavy pole index or -1."""
    passes = 0
    if j < K - 1:
        de = kd[j + 1] - kd[j]
        mid = 0.5 * de
        terms = kz2 / ((kd - kd[j]) - mid)
        s = np.sum(terms); passes += 1
        if 1.0 + rho * s >= 0.0:
            o, lo, hi = j, 0.0, mid
        else:
            o, lo, hi = j + 1, -mid, 0.0
        dorg = kd[o]
        tau = 0.5 * (lo + hi)
        C = 1.0 / rho + s + kz2[j] / mid - kz2[j + 1] / mid
        heavy = h >= 0 and h != j and h != j + 1
        if heavy:
            C -= terms[h]
            ph = kd[h] - dorg
        x = tau
        g = None
        for _ in range(nfix if heavy else 1):
            ce = C + (kz2[h] / (ph - x) if heavy else 0.0)
            g = quad_origin_lo(ce, kz2[j], kz2[j + 1], de) if o == j else quad_origin_hi(ce, kz2[j], kz2[j + 1], de)
            if not (lo < g < hi):
                break
            x = g
        if g is not None and lo < g < hi:
            tau = g
    else:
        o, lo, hi = j, 0.0, rho * sumz2 * (1.0 + 4.0 * EPS)
        dorg = kd[o]
        tau = 0.5 * (lo + hi)
        if K >= 2:
            heavy = h >= 0 and h < K - 2
            msk = np.ones(K, bool); msk[K - 2:] = False
            if heavy:
                msk[h] = False
            sm = np.sum(kz2[msk] / (kd[msk] - kd[K - 1])); passes += 1
            C = 1.0 / rho + sm; dl = kd[K - 2] - kd[K - 1]; a = kz2[K - 2]; b = kz2[K - 1]
            ph = (kd[h] - dorg) if heavy else 0.0
            x = 0.0
            g = None
            for _ in range(nfix if heavy else 1):
                ce = C + (kz2[h] / (ph - x) if heavy else 0.0)
                if ce > 0:
                    Bm = ce * dl + a + b
                    sq = np.sqrt(max(Bm * Bm - 4.0 * ce * b * dl, 0.0))
                    g = (Bm + sq) / (2.0 * ce) if Bm > 0 else (2.0 * b * dl) / (Bm - sq)
                    if not (lo < g < hi):
                        break
                    x = g
                else:
                    g = None
                    break
            if g is not None and lo < g < hi:
                tau = g
    it = 0
    idx = np.arange(K)
    heavy_i = h >= 0 and h != j and not (j < K - 1 and h == j + 1)
    while it < 120:
        rdel = 1.0 / ((kd - dorg) - tau)
        t = kz2 * rdel
        dt = t * rdel
        passes += 1
        th = dth = 0.0
        if heavy_i:
            th = rho * t[h]; dth = rho * dt[h]
        psi = rho * np.sum(t[idx <= j]); phi = rho * np.sum(t[idx > j])
        dpsi = rho * np.sum(dt[idx <= j]); dphi = rho * np.sum(dt[idx > j])
        aerr = rho * np.sum(np.abs(t))
        f = 1.0 + psi + phi
        if trace:
            print("   it", it, "tau", tau, "f", f, "lo", lo, "hi", hi)
        if f < 0:
            lo = max(lo, tau)
        else:
            hi = min(hi, tau)
        if abs(f) <= 4.0 * EPS * K * (1.0 + aerr):
            break
        # heavy pole out of its side's sums
        if heavy_i:
            if h <= j:
                psi -= th; dpsi -= dth
            else:
                phi -= th; dphi -= dth
            Dh = (kd[h] - dorg) - tau
            sh = rho * kz2[h]
        D1 = (kd[j] - dorg) - tau
        ok = False
        nt = 0.0
        if j < K - 1:
            D2 = (kd[j + 1] - dorg) - tau
            q1 = dpsi * D1 * D1; q2 = dphi * D2 * D2
            c = 1.0 + psi - dpsi * D1 + phi - dphi * D2
            eta = 0.0
            for _ in range(nfix if heavy_i else 1):
                ce = c + (sh / (Dh - eta) if heavy_i else 0.0)
                Bq = ce * (D1 + D2) + q1 + q2
                Cq = D1 * D2 * (ce + q1 / D1 + q2 / D2) if heavy_i else D1 * D2 * f
                disc = Bq * Bq - 4.0 * ce * Cq
                if disc < 0:
                    ok = False
                    break
                sq = np.sqrt(disc)
                den = Bq + (sq if Bq >= 0 else -sq)
                if den == 0:
                    ok = False
                    break
                eta = 2.0 * Cq / den
                ok = True
                if not (lo < tau + eta < hi):
                    break
            nt = tau + eta
        else:
            # last root: 1 + heavy (exact) + one floating effective pole for the rest
            Pv = -(psi + phi); dP = dpsi + dphi   # rest: Pv = s/(eta - D*)... all poles below
            if Pv > 0 and dP > 0:
                if heavy_i:
                    # rest(eta) = -Pv^2/dP / (Pv/dP + eta)   [value -Pv, derivative dP at eta = 0]
                    sr = Pv * Pv / dP; Dr = -Pv / dP      # rest = sr / (Dr - eta), Dr < 0
                    # 1 + sh/(Dh - eta) + sr/(Dr - eta) = 0, both poles below: eta > max(Dh, Dr)
                    # (Dh-eta)(Dr-eta) + sh (Dr-eta) + sr (Dh-eta) = 0
                    # eta^2 - (Dh + Dr + sh + sr) eta + Dh Dr + sh Dr + sr Dh = 0  -> larger root
                    Bm = Dh + Dr + sh + sr
                    Cm = Dh * Dr + sh * Dr + sr * Dh
                    disc = Bm * Bm - 4.0 * Cm
                    if disc >= 0:
                        sq = np.sqrt(disc)
                        eta = 0.5 * (Bm + sq) if Bm > 0 else 2.0 * Cm / (Bm - sq)
                        nt = tau + eta
                        ok = True
                else:
                    nt = tau + (Pv * Pv - Pv) / dP
                    ok = True
        if (not ok) or not (lo < nt < hi):
            pos = hi > 0
            a = max(lo if pos else -hi, 4.0 * EPS * max(abs(dorg), 1e-300)); b = hi if pos else -lo
            if b > 1e9 * a:
                nt = np.sqrt(a * b) if pos else -np.sqrt(a * b)
            else:
                nt = 0.5 * (lo + hi)
            if trace:
                print("     safeguard ->", nt)
        if nt == tau or hi - lo <= 2.0 * EPS * max(abs(lo), abs(hi)):
            tau = nt
            break
        tau = nt
        it += 1
    return tau, o, it, passes


if __name__ == "__main__":
    P = np.load(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/secular_problems.npy")
    nprob = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    nfix = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    allold, allnew, mxo, mxn, maxdiff = [], [], [], [], 0.0
    for pi in range(min(nprob, len(P))):
        o = P[pi]; K = int(o[0])
        if K == 0:
            continue
        rho = o[1]; kd = o[8:8 + K].copy(); kz2 = o[268:268 + K].copy()
        h = int(np.argmax(kz2))
        if kz2[h] < 0.5 * o[2]:
            h = -1
        old = [root_old(kd, kz2, K, rho, o[2], j) for j in range(K)]
        new = [root(kd, kz2, K, rho, o[2], j, h, nfix) for j in range(K)]
        io = np.array([r[2] for r in old]); inn = np.array([r[2] for r in new])
        for j in range(K):
            lo_ = kd[old[j][1]] + old[j][0]; ln_ = kd[new[j][1]] + new[j][0]
            # compare tau relative to distance to the origin pole when same origin
            if old[j][1] == new[j][1]:
                rel = abs(old[j][0] - new[j][0]) / max(abs(old[j][0]), 1e-300)
            else:
                rel = abs(lo_ - ln_) / max(abs(lo_), 1e-300)
            maxdiff = max(maxdiff, rel)
        allold.append(io); allnew.append(inn); mxo.append(io.max()); mxn.append(inn.max())
    allold = np.concatenate(allold); allnew = np.concatenate(allnew)
    print("old: mean its %.3f, max-per-problem mean %.2f max %d; hist %s" % (allold.mean(), np.mean(mxo), max(mxo), np.bincount(allold)))
    print("new: mean its %.3f, max-per-problem mean %.2f max %d; hist %s" % (allnew.mean(), np.mean(mxn), max(mxn), np.bincount(allnew)))
    print("max rel diff of tau between schemes: %.2e" % maxdiff)
    print("per-problem max (old,new):", list(zip(mxo, mxn))[:40])
