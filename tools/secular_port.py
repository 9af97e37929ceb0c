"""Dev helper: Python port of event_kernel.cu's secular_root (same arithmetic
up to summation order) run over dumped problems (tools/dump_secular.py), to
study iteration counts of alternative initial guesses / iterations offline."""
import sys
import numpy as np

EPS = np.finfo(np.float64).eps


def root(kd, kz2, K, rho, sumz2, j, variant=0, trace=False):
    if j < K - 1:
        mid = 0.5 * (kd[j + 1] - kd[j])
        s = np.sum(kz2 / ((kd - kd[j]) - mid))
        if 1.0 + rho * s >= 0.0:
            o, lo, hi = j, 0.0, mid
        else:
            o, lo, hi = j + 1, -mid, 0.0
    else:
        o, lo, hi = j, 0.0, rho * sumz2 * (1.0 + 4.0 * EPS)
    dorg = kd[o]
    tau = 0.5 * (lo + hi)
    if j < K - 1:
        de = kd[j + 1] - kd[j]
        mid = 0.5 * de
        sm = s
        C = 1.0 / rho + sm + kz2[j] / mid - kz2[j + 1] / mid
        if variant & 1:
            # background evaluated at the origin pole instead of the midpoint
            oth = np.ones(K, bool); oth[j] = False; oth[j + 1] = False
            C = 1.0 / rho + np.sum(kz2[oth] / (kd[oth] - dorg))
        if o == j:
            Aq = C * de + kz2[j] + kz2[j + 1]; Bq = kz2[j] * de
            sq = np.sqrt(abs(Aq * Aq - 4.0 * Bq * C))
            g = 2.0 * Bq / (Aq + sq) if Aq > 0 else (Aq - sq) / (2.0 * C)
        else:
            Aq = C * de - kz2[j] - kz2[j + 1]; Bq = kz2[j + 1] * de
            sq = np.sqrt(abs(Aq * Aq + 4.0 * Bq * C))
            g = 2.0 * Bq / (Aq - sq) if Aq < 0 else -(Aq + sq) / (2.0 * C)
        if lo < g < hi:
            tau = g
    elif K >= 2:
        sm = np.sum(kz2[:K - 2] / (kd[:K - 2] - kd[K - 1]))
        C = 1.0 / rho + sm; dl = kd[K - 2] - kd[K - 1]; a = kz2[K - 2]; b = kz2[K - 1]
        if C > 0:
            Bm = C * dl + a + b
            sq = np.sqrt(max(Bm * Bm - 4.0 * C * b * dl, 0.0))
            g = (Bm + sq) / (2.0 * C) if Bm > 0 else (2.0 * b * dl) / (Bm - sq)
            if lo < g < hi:
                tau = g
    it = 0
    idx = np.arange(K)
    while it < 120:
        rdel = 1.0 / ((kd - dorg) - tau)
        t = kz2 * rdel
        dt = t * rdel
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
        D1 = (kd[j] - dorg) - tau
        ok = False
        nt = 0.0
        if j < K - 1:
            D2 = (kd[j + 1] - dorg) - tau
            q1 = dpsi * D1 * D1; q2 = dphi * D2 * D2
            c = 1.0 + psi - dpsi * D1 + phi - dphi * D2
            Bq = c * (D1 + D2) + q1 + q2
            Cq = D1 * D2 * f
            disc = Bq * Bq - 4.0 * c * Cq
            if disc >= 0:
                sq = np.sqrt(disc)
                den = Bq + (sq if Bq >= 0 else -sq)
                if den != 0:
                    nt = tau + 2.0 * Cq / den
                    ok = True
        else:
            Pv = -(psi + phi); dP = dpsi + dphi
            if Pv > 0 and dP > 0:
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
    return tau, o, it


if __name__ == "__main__":
    P = np.load(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/secular_problems.npy")
    variant = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    nprob = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    mism = 0
    mx = []
    for pi in range(min(nprob, len(P))):
        o = P[pi]; K = int(o[0])
        if K == 0:
            continue
        rho = o[1]; kd = o[8:8 + K].copy(); kz2 = o[268:268 + K].copy(); its = o[530:530 + K].astype(int)
        mine = np.array([root(kd, kz2, K, rho, o[2], j, variant)[2] for j in range(K)])
        mism += int(np.sum(mine != its))
        mx.append((its.max(), mine.max(), int(np.argmax(mine))))
    print("variant", variant, "mismatching counts vs device:", mism)
    print("max its per problem (device, port, argmax):", mx)
