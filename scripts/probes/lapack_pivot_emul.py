"""Which arithmetic decides LAPACK dgeqp3's pivots on the WQ moment systems?
Emulates dgeqp3 -> dlaqp2 (unblocked: min(t,m) < NB) in Python, with each
BLAS call either the exact OpenBLAS routine (scipy.linalg.blas) or a plain
restatement, and compares the pivots with scipy.linalg.qr(pivoting=True).
Development probe for the GPU fit kernel; CPU only."""
import sys, os, itertools
sys.path.insert(0, os.getcwd())
import numpy as np
import scipy.linalg
from scipy.linalg import blas
from oracle import bspline as B, quad as Q

EPS = np.finfo(float).eps
TOL3Z = np.sqrt(EPS)


def systems(nel, p):
    sp_ = B.uniform_space(nel, p)
    lay = Q.place_wq_points(sp_)
    M = Q.mass_1d(sp_)
    f, V = sp_.eval_nonzero(lay.points)
    out = []
    for i in range(sp_.n):
        k0, k1 = lay.range_for(sp_.el_first[i], sp_.el_last[i])
        j0, j1 = int(sp_.ov_lo[i]), int(sp_.ov_hi[i])
        A = np.zeros((j1 - j0 + 1, k1 - k0))
        for r in range(p + 1):
            jj = f[k0:k1] + r - j0
            ok = (jj >= 0) & (jj <= j1 - j0)
            A[jj[ok], np.nonzero(ok)[0]] = V[k0:k1][ok, r]
        out.append((A, M[i, j0:j1 + 1]))
    return out


def nrm2_exact(x):
    import math
    return math.sqrt(math.fsum(float(v) * float(v) for v in x)) if len(x) else 0.0


def nrm2_exact_cr(x):
    from fractions import Fraction
    import math
    s = sum(Fraction(float(v)) ** 2 for v in x)
    r = math.sqrt(float(s))
    # correct rounding of sqrt(s)
    best = r
    for cand in (np.nextafter(r, 0), r, np.nextafter(r, np.inf)):
        if abs(Fraction(float(cand)) ** 2 - s) < abs(Fraction(float(best)) ** 2 - s):
            best = float(cand)
    return best


def dlapy2(x, y):
    xa, ya = abs(x), abs(y)
    w, z = max(xa, ya), min(xa, ya)
    return w if z == 0.0 else w * np.sqrt(1.0 + (z / w) ** 2)


def emulate(A, nrm="blas", gemv="blas", ger="blas"):
    A = np.asfortranarray(A.copy())
    t, m = A.shape
    norm = {"blas": lambda x: blas.dnrm2(x) if x.size else 0.0, "fsum": nrm2_exact,
            "cr": nrm2_exact_cr, "naive": lambda x: float(np.sqrt(np.sum(x * x))),
            "seq": lambda x: float(np.sqrt(sum(float(v) * float(v) for v in x)))}[nrm]
    jpvt = np.arange(m)
    vn1 = np.array([norm(A[:, j]) for j in range(m)])
    vn2 = vn1.copy()
    mn = min(t, m)
    for i in range(mn):
        pvt = i + int(np.argmax(np.abs(vn1[i:])))          # idamax: first max
        if pvt != i:
            A[:, [i, pvt]] = A[:, [pvt, i]]
            jpvt[[i, pvt]] = jpvt[[pvt, i]]
            vn1[pvt], vn2[pvt] = vn1[i], vn2[i]
        # dlarfg(t-i, A[i,i], A[i+1:,i])
        alpha = A[i, i]
        x = A[i + 1:, i]
        xnorm = norm(x) if x.size else 0.0
        if xnorm == 0.0:
            tau = 0.0
        else:
            beta = -np.copysign(dlapy2(alpha, xnorm), alpha)
            tau = (beta - alpha) / beta
            A[i + 1:, i] = x * (1.0 / (alpha - beta)) if gemv != "blas" else blas.dscal(1.0 / (alpha - beta), x.copy())
            A[i, i] = beta
        if i < m - 1 and tau != 0.0:
            v = np.concatenate([[1.0], A[i + 1:, i]])
            C = A[i:, i + 1:]
            if gemv == "blas":
                w = blas.dgemv(1.0, np.asfortranarray(C), v, trans=1)
            else:
                w = np.array([sum(C[r, c] * v[r] for r in range(v.size)) for c in range(C.shape[1])])
            if ger == "blas":
                A[i:, i + 1:] = blas.dger(-tau, v, w, a=np.asfortranarray(C))
            else:
                A[i:, i + 1:] = C - tau * np.outer(v, w)
        for j in range(i + 1, m):
            if vn1[j] != 0.0:
                temp = 1.0 - (abs(A[i, j]) / vn1[j]) ** 2
                temp = max(temp, 0.0)
                temp2 = temp * (vn1[j] / vn2[j]) ** 2
                if temp2 <= TOL3Z:
                    if i < t - 1:
                        vn1[j] = norm(A[i + 1:, j])
                        vn2[j] = vn1[j]
                    else:
                        vn1[j] = vn2[j] = 0.0
                else:
                    vn1[j] = vn1[j] * np.sqrt(temp)
    return jpvt


if __name__ == "__main__" and "more" not in sys.argv and "which" not in sys.argv and "which2" not in sys.argv and "which3" not in sys.argv and "solve" not in sys.argv and "one" not in sys.argv and "qtb" not in sys.argv and "parts" not in sys.argv and "tails" not in sys.argv and "dbg" not in sys.argv and "dbg2" not in sys.argv and "dbg3" not in sys.argv:
    cases = [(9, 1), (9, 2), (9, 3), (7, 4), (8, 5), (10, 6), (16, 2), (64, 3), (12, 8), (40, 6), (40, 8)]
    variants = [("blas", "blas", "blas"), ("fsum", "blas", "blas"), ("cr", "blas", "blas"),
                ("naive", "blas", "blas"), ("seq", "blas", "blas"), ("cr", "seq", "seq"), ("seq", "seq", "seq")]
    tot = {v: 0 for v in variants}
    n = 0
    for nel, p in cases:
        for A, b in systems(nel, p):
            _, _, piv = scipy.linalg.qr(A, mode="economic", pivoting=True)
            n += 1
            for v in variants:
                jp = emulate(A, *v)
                r = min(A.shape)
                tot[v] += int(np.array_equal(jp[:r], piv[:r]))
    for v in variants:
        print(v, f"{tot[v]}/{n}")


def dd_norm(x):
    """The GPU algorithm: squares summed in double-double (TwoProd by fma,
    TwoSum), then a correctly rounded sqrt of the double-double."""
    import math
    from fractions import Fraction as F

    def fma(a, b, c):          # one rounding of a*b + c (what the GPU's fma does)
        return float(F(a) * F(b) + F(c))
    hi = lo = 0.0
    for v in x:
        v = float(v)
        p = v * v
        pe = fma(v, v, -p)
        s = hi + p
        bb = s - hi
        err = (hi - (s - bb)) + (p - bb)
        hi, lo = s, lo + err + pe
    s = hi + lo
    lo = lo - (s - hi)
    hi = s
    if hi <= 0.0:
        return 0.0
    r = math.sqrt(hi)
    e = fma(-r, r, hi) + lo
    up = np.nextafter(r, np.inf)
    u = up - r
    if e - r * u > 0.25 * u * u:
        return float(up)
    dn = np.nextafter(r, 0.0)
    d = r - dn
    if -e - r * d > -0.25 * d * d:
        return float(dn)
    return r


CASES_REC = [(9, 1), (9, 2), (9, 3), (7, 4), (8, 5), (10, 6), (16, 2), (12, 8), (24, 7), (20, 8)]
if "wide" in sys.argv:
    CASES_REC = CASES_REC + [(32, 4), (48, 6), (30, 8), (17, 5), (33, 3), (64, 4)]


def recorded_systems():
    """Every moment system the oracle solves while building WQ and DWQ rules
    for a range of spaces, uniform and non-uniform."""
    rec = []
    orig = Q.qr_basic

    def spy(A, b):
        rec.append((A.copy(), b.copy()))
        return orig(A, b)
    Q.qr_basic = spy
    try:
        for nel, p in CASES_REC:
            sp_ = B.uniform_space(nel, p)
            lay = Q.place_wq_points(sp_)
            Q.compute_wq_rules(sp_, lay)
            for u in (sp_.bp[nel // 2], sp_.bp[nel // 3], sp_.bp[1]):
                try:
                    Q.build_dwq(sp_, lay, float(u))
                except Exception as exc:
                    print("dwq skip", nel, p, u, exc)
        kn = np.array([0, 0, 0, 0.1, 0.25, 0.25, 0.5, 0.5, 0.5, 0.8, 1, 1, 1.0])
        sp_ = B.Space1D(kn, 2)
        Q.compute_wq_rules(sp_, Q.place_wq_points(sp_))
    finally:
        Q.qr_basic = orig
    return rec


def main2():
    rec = recorded_systems()
    variants = {"blas": ("blas", "blas", "blas"), "cr/seq": ("cr", "seq", "seq")}
    ok = {k: 0 for k in variants}
    ok["dd/seq"] = 0
    norms_equal = 0
    nn = 0
    for A, b in rec:
        _, _, piv = scipy.linalg.qr(A, mode="economic", pivoting=True)
        r = min(A.shape)
        for k, v in variants.items():
            ok[k] += int(np.array_equal(emulate(A, *v)[:r], piv[:r]))
        for j in range(A.shape[1]):
            nn += 1
            norms_equal += dd_norm(A[:, j]) == nrm2_exact_cr(A[:, j])
    global nrm2_dd
    print({k: f"{v}/{len(rec)}" for k, v in ok.items() if k != "dd/seq"}, f"dd==cr norms {norms_equal}/{nn}")


if __name__ == "__main__" and "more" in sys.argv and "which" not in sys.argv and "which2" not in sys.argv and "which3" not in sys.argv and "solve" not in sys.argv and "one" not in sys.argv and "qtb" not in sys.argv and "parts" not in sys.argv and "tails" not in sys.argv and "dbg" not in sys.argv and "dbg2" not in sys.argv and "dbg3" not in sys.argv:
    main2()


def main3():
    rec = recorded_systems()
    variants = [("cr", "blas", "blas"), ("cr", "seq", "blas"), ("cr", "blas", "seq"), ("cr", "seq", "seq")]
    bad = {v: [] for v in variants}
    for n, (A, b) in enumerate(rec):
        _, _, piv = scipy.linalg.qr(A, mode="economic", pivoting=True)
        r = min(A.shape)
        for v in variants:
            if not np.array_equal(emulate(A, *v)[:r], piv[:r]):
                bad[v].append(n)
    for v in variants:
        print(v, len(bad[v]), bad[v][:10])
    return rec, bad


if __name__ == "__main__" and "which" in sys.argv and "which2" not in sys.argv and "which3" not in sys.argv and "solve" not in sys.argv and "one" not in sys.argv and "qtb" not in sys.argv and "parts" not in sys.argv and "tails" not in sys.argv and "dbg" not in sys.argv and "dbg2" not in sys.argv and "dbg3" not in sys.argv:
    main3()


def _fma(a, b, c):
    from fractions import Fraction as F
    return float(F(float(a)) * F(float(b)) + F(float(c)))


def gemv_t(C, v, kind):
    out = np.zeros(C.shape[1])
    for c in range(C.shape[1]):
        col = C[:, c]
        if kind == "seq":
            acc = 0.0
            for r in range(v.size):
                acc = acc + col[r] * v[r]
        elif kind == "seqfma":
            acc = 0.0
            for r in range(v.size):
                acc = _fma(col[r], v[r], acc)
        elif kind.startswith("fma"):
            L = int(kind[3:])
            part = [0.0] * L
            n4 = (v.size // L) * L
            for r in range(n4):
                part[r % L] = _fma(col[r], v[r], part[r % L])
            acc = 0.0
            while len(part) > 1:
                part = [part[2 * q] + part[2 * q + 1] for q in range(len(part) // 2)]
            acc = part[0]
            for r in range(n4, v.size):
                acc = _fma(col[r], v[r], acc)
        out[c] = acc
    return out


def ger(C, tau, v, w, kind):
    C = C.copy()
    for j in range(C.shape[1]):
        temp = -tau * w[j]
        for i in range(v.size):
            C[i, j] = _fma(v[i], temp, C[i, j]) if kind == "reffma" else C[i, j] + v[i] * temp
    return C


def emulate2(A, gk, rk):
    A = np.asfortranarray(A.copy())
    t, m = A.shape
    norm = nrm2_exact_cr
    jpvt = np.arange(m)
    vn1 = np.array([norm(A[:, j]) for j in range(m)])
    vn2 = vn1.copy()
    for i in range(min(t, m)):
        pvt = i + int(np.argmax(np.abs(vn1[i:])))
        if pvt != i:
            A[:, [i, pvt]] = A[:, [pvt, i]]
            jpvt[[i, pvt]] = jpvt[[pvt, i]]
            vn1[pvt], vn2[pvt] = vn1[i], vn2[i]
        alpha = A[i, i]
        x = A[i + 1:, i]
        xnorm = norm(x) if x.size else 0.0
        tau = 0.0
        if xnorm != 0.0:
            beta = -np.copysign(dlapy2(alpha, xnorm), alpha)
            tau = (beta - alpha) / beta
            A[i + 1:, i] = x * (1.0 / (alpha - beta))
            A[i, i] = beta
        if i < m - 1 and tau != 0.0:
            v = np.concatenate([[1.0], A[i + 1:, i]])
            lastv = v.size
            while lastv > 0 and v[lastv - 1] == 0.0:          # dlarf: last non-zero of v
                lastv -= 1
            C = A[i:i + lastv, i + 1:]
            nz = np.nonzero(np.any(C != 0.0, axis=0))[0]
            lastc = int(nz[-1]) + 1 if nz.size else 0         # iladlc
            if lastv and lastc:
                Cs = C[:, :lastc]
                vv = v[:lastv]
                w = gemv_t(Cs, vv, gk) if gk != "blas" else blas.dgemv(1.0, np.asfortranarray(Cs), vv, trans=1)
                A[i:i + lastv, i + 1:i + 1 + lastc] = (ger(Cs, tau, vv, w, rk) if rk != "blas"
                                                       else blas.dger(-tau, vv, w, a=np.asfortranarray(Cs)))
        for j in range(i + 1, m):
            if vn1[j] != 0.0:
                temp = max(1.0 - (abs(A[i, j]) / vn1[j]) ** 2, 0.0)
                if temp * (vn1[j] / vn2[j]) ** 2 <= TOL3Z:
                    vn1[j] = norm(A[i + 1:, j]) if i < t - 1 else 0.0
                    vn2[j] = vn1[j]
                else:
                    vn1[j] = vn1[j] * np.sqrt(temp)
    return jpvt


if __name__ == "__main__" and "which2" in sys.argv and "which3" not in sys.argv and "solve" not in sys.argv and "one" not in sys.argv and "qtb" not in sys.argv and "parts" not in sys.argv and "tails" not in sys.argv and "dbg" not in sys.argv and "dbg2" not in sys.argv and "dbg3" not in sys.argv:
    rec = recorded_systems()
    idx = [127, 333, 334, 335, 336, 337, 338, 339]
    sub = [rec[k] for k in idx]
    print("shapes", [a.shape for a, _ in sub])
    for gk in ("blas", "seq", "seqfma", "fma2", "fma4"):
        for rk in ("blas", "ref", "reffma"):
            n = 0
            for A, b in sub:
                _, _, piv = scipy.linalg.qr(A, mode="economic", pivoting=True)
                r = min(A.shape)
                n += np.array_equal(emulate2(A, gk, rk)[:r], piv[:r])
            print(gk, rk, f"{n}/{len(sub)}", flush=True)


def gemv_ob(C, v, variant):
    """OpenBLAS-style dgemv_t guesses: rows in blocks of 4 with 4 FMA lane
    accumulators, reduced, then the m % 4 leftover rows as one expression."""
    m = v.size
    m1 = m - m % 4
    out = np.zeros(C.shape[1])
    for c in range(C.shape[1]):
        col = C[:, c]
        p = [0.0] * 4
        for r in range(m1):
            p[r % 4] = _fma(col[r], v[r], p[r % 4])
        if variant[0] == "a":
            dot = (p[0] + p[1]) + (p[2] + p[3])
        else:
            dot = (p[0] + p[2]) + (p[1] + p[3])
        y = 0.0 + dot
        lo = [(col[r], v[r]) for r in range(m1, m)]
        if lo:
            if variant[1] == "f":           # fma chain over the leftover products
                t = lo[0][0] * lo[0][1]
                for a, x in lo[1:]:
                    t = _fma(a, x, t)
                y = y + t
            elif variant[1] == "g":         # fully contracted into y
                for a, x in lo:
                    y = _fma(a, x, y)
            else:                            # plain products and adds
                t = lo[0][0] * lo[0][1]
                for a, x in lo[1:]:
                    t = t + a * x
                y = y + t
        out[c] = y
    return out


if __name__ == "__main__" and "which3" in sys.argv:
    rec = recorded_systems()
    for variant in (("bp",) if "wide" in sys.argv else ("af", "ag", "ap", "bf", "bg", "bp")):
        bad = 0
        for A, b in rec:
            _, _, piv = scipy.linalg.qr(A, mode="economic", pivoting=True)
            r = min(A.shape)
            gemv_t_saved = globals()["gemv_t"]
            globals()["gemv_t"] = lambda C, v, k, _v=variant: gemv_ob(C, v, _v)
            ok = np.array_equal(emulate2(A, "x", "reffma")[:r], piv[:r])
            globals()["gemv_t"] = gemv_t_saved
            bad += not ok
        print(variant, "mismatches", bad, "of", len(rec), flush=True)


def solve_emul(A, b):
    """emulate2's factorisation + the GPU kernel's solve (reflectors applied
    to b with the same dlarf arithmetic, back substitution) -> (w, piv, rank)."""
    A = np.asfortranarray(A.copy())
    bb = b.copy()
    t, m = A.shape
    norm = nrm2_exact_cr
    jpvt = np.arange(m)
    vn1 = np.array([norm(A[:, j]) for j in range(m)])
    vn2 = vn1.copy()
    for i in range(min(t, m)):
        pvt = i + int(np.argmax(np.abs(vn1[i:])))
        if pvt != i:
            A[:, [i, pvt]] = A[:, [pvt, i]]
            jpvt[[i, pvt]] = jpvt[[pvt, i]]
            vn1[pvt], vn2[pvt] = vn1[i], vn2[i]
        alpha = A[i, i]
        x = A[i + 1:, i]
        xnorm = norm(x) if x.size else 0.0
        tau = 0.0
        if xnorm != 0.0:
            beta = -np.copysign(dlapy2(alpha, xnorm), alpha)
            tau = (beta - alpha) / beta
            A[i + 1:, i] = x * (1.0 / (alpha - beta))
            A[i, i] = beta
        v = np.concatenate([[1.0], A[i + 1:, i]])
        lastv = v.size
        while lastv > 0 and v[lastv - 1] == 0.0:
            lastv -= 1
        if tau != 0.0:
            for c in list(range(i + 1, m)) + ["b"]:
                col = bb[i:i + lastv] if c == "b" else A[i:i + lastv, c]
                w = gemv_ob(col[:, None], v[:lastv], "bp")[0]
                temp = -tau * w
                newc = np.array([_fma(v[r], temp, col[r]) for r in range(lastv)])
                if c == "b":
                    bb[i:i + lastv] = newc
                else:
                    A[i:i + lastv, c] = newc
        for j in range(i + 1, m):
            if vn1[j] != 0.0:
                temp = max(1.0 - (abs(A[i, j]) / vn1[j]) ** 2, 0.0)
                if temp * (vn1[j] / vn2[j]) ** 2 <= TOL3Z:
                    vn1[j] = norm(A[i + 1:, j]) if i < t - 1 else 0.0
                    vn2[j] = vn1[j]
                else:
                    vn1[j] = vn1[j] * np.sqrt(temp)
    d = np.abs(np.diag(A[:min(t, m), :min(t, m)]))
    thr = max(t, m) * EPS * d[0]
    rank = int(np.sum(d > thr))
    z = np.zeros(rank)
    for k in range(rank - 1, -1, -1):
        acc = bb[k]
        for c in range(k + 1, rank):
            acc -= A[k, c] * z[c]
        z[k] = acc / A[k, k]
    w = np.zeros(m)
    w[jpvt[:rank]] = z
    return w, jpvt, rank


if __name__ == "__main__" and "solve" in sys.argv:
    for nel, p in [(12, 8), (10, 6), (8, 5), (7, 4), (9, 2)]:
        for A, b in systems(nel, p):
            Q_, R, piv = scipy.linalg.qr(A, mode="economic", pivoting=True)
            wref = Q.qr_basic(A, b)
            w, jp, rank = solve_emul(A, b)
            r = min(A.shape)
            d = np.abs(np.diag(R))
            rref = int(np.sum(d > max(A.shape) * EPS * d[0]))
            same_piv = np.array_equal(jp[:r], piv[:r])
            err = np.max(np.abs(w - wref)) / np.max(np.abs(wref))
            if not same_piv or err > 1e-12 or rank != rref:
                print(nel, p, A.shape, "piv same", same_piv, "rank", rank, rref, f"w err {err:.2e}",
                      "cond", f"{d[0] / d[rref - 1]:.2e}")


if __name__ == "__main__" and "one" in sys.argv:
    nel, p = int(sys.argv[2]), int(sys.argv[3])
    for i, (A, b) in enumerate(systems(nel, p)):
        _, R, piv = scipy.linalg.qr(A, mode="economic", pivoting=True)
        w, jp, rank = solve_emul(A, b)
        wref = Q.qr_basic(A, b)
        r = min(A.shape)
        err = np.max(np.abs(w - wref)) / np.max(np.abs(wref))
        if not np.array_equal(jp[:r], piv[:r]) or err > 1e-12:
            print(i, A.shape, "emul piv", jp[:r], "lapack", piv[:r], f"err {err:.1e}")
    print("done")


def factor_emul(A):
    """-> (A with R above the diagonal and reflectors below, tau, jpvt) as dlaqp2."""
    A = np.asfortranarray(A.copy())
    t, m = A.shape
    norm = nrm2_exact_cr
    jpvt = np.arange(m)
    tau_all = np.zeros(min(t, m))
    vn1 = np.array([norm(A[:, j]) for j in range(m)])
    vn2 = vn1.copy()
    for i in range(min(t, m)):
        pvt = i + int(np.argmax(np.abs(vn1[i:])))
        if pvt != i:
            A[:, [i, pvt]] = A[:, [pvt, i]]
            jpvt[[i, pvt]] = jpvt[[pvt, i]]
            vn1[pvt], vn2[pvt] = vn1[i], vn2[i]
        alpha = A[i, i]
        x = A[i + 1:, i]
        xnorm = norm(x) if x.size else 0.0
        tau = 0.0
        if xnorm != 0.0:
            beta = -np.copysign(dlapy2(alpha, xnorm), alpha)
            tau = (beta - alpha) / beta
            A[i + 1:, i] = x * (1.0 / (alpha - beta))
            A[i, i] = beta
        tau_all[i] = tau
        if tau != 0.0 and i < m - 1:
            v = np.concatenate([[1.0], A[i + 1:, i]])
            apply_h(A[i:, i + 1:], v, tau)
        for j in range(i + 1, m):
            if vn1[j] != 0.0:
                temp = max(1.0 - (abs(A[i, j]) / vn1[j]) ** 2, 0.0)
                if temp * (vn1[j] / vn2[j]) ** 2 <= TOL3Z:
                    vn1[j] = norm(A[i + 1:, j]) if i < t - 1 else 0.0
                    vn2[j] = vn1[j]
                else:
                    vn1[j] = vn1[j] * np.sqrt(temp)
    return A, tau_all, jpvt


def apply_h(C, v, tau):
    """dlarf('Left') in place on C (rows = v's length): lastv/lastc trims,
    'bp' dgemv_t, FMA dger."""
    lastv = v.size
    while lastv > 0 and v[lastv - 1] == 0.0:
        lastv -= 1
    if lastv == 0:
        return
    for c in range(C.shape[1]):
        col = C[:lastv, c]
        if not np.any(col != 0.0):
            continue
        w = gemv_ob(col[:, None], v[:lastv], "bp")[0]
        temp = -tau * w
        C[:lastv, c] = [_fma(v[r], temp, col[r]) for r in range(lastv)]


def dorg2r(Af, tau, n):
    t = Af.shape[0]
    k = n
    Qm = np.asfortranarray(np.zeros((t, n)))
    Qm[:, :k] = Af[:, :k]
    for j in range(k, n):
        Qm[:, j] = 0.0
        Qm[j, j] = 1.0
    for i in range(k - 1, -1, -1):
        if i < n - 1:
            Qm[i, i] = 1.0
            v = Qm[i:, i].copy()
            apply_h(Qm[i:, i + 1:], v, tau[i])
        if i < t - 1:
            Qm[i + 1:, i] = Qm[i + 1:, i] * (-tau[i])
        Qm[i, i] = 1.0 - tau[i]
        Qm[:i, i] = 0.0
    return Qm


def solve_emul2(A, b, recip):
    t, m = A.shape
    Af, tau, jp = factor_emul(A)
    n = min(t, m)
    Qm = dorg2r(Af, tau, n)
    y = gemv_ob(Qm, b, "bp")
    R = np.triu(Af[:n, :n])
    d = np.abs(np.diag(R))
    rank = int(np.sum(d > max(t, m) * EPS * d[0]))
    z = np.zeros(rank)
    for k in range(rank - 1, -1, -1):
        acc = y[k]
        for c in range(k + 1, rank):
            acc -= R[k, c] * z[c]
        z[k] = acc * (1.0 / R[k, k]) if recip else acc / R[k, k]
    w = np.zeros(m)
    w[jp[:rank]] = z
    return w


if __name__ == "__main__" and "qtb" in sys.argv:
    for recip in (False, True):
        errs = []
        for A, b in systems(12, 8) + systems(10, 6):
            wref = Q.qr_basic(A, b)
            w = solve_emul2(A, b, recip)
            errs.append(np.max(np.abs(w - wref)) / np.max(np.abs(wref)))
        errs = np.array(errs)
        print("recip", recip, "exact", int((errs == 0).sum()), "of", errs.size, "max err", errs.max())


if __name__ == "__main__" and "parts" in sys.argv:
    nR = nQ = ny = nz = 0
    S = systems(12, 8) + systems(10, 6) + systems(9, 3)
    for A, b in S:
        Qs, Rs, piv = scipy.linalg.qr(A, mode="economic", pivoting=True)
        t, m = A.shape
        n = min(t, m)
        Af, tau, jp = factor_emul(A)
        R = np.triu(Af[:n, :])
        nR += np.array_equal(R, Rs)
        Qm = dorg2r(Af, tau, n)
        nQ += np.array_equal(Qm, Qs)
        y = gemv_ob(Qs, b, "bp")
        ny += np.array_equal(y, Qs.T @ b)
        d = np.abs(np.diag(Rs))
        rank = int(np.sum(d > max(t, m) * EPS * d[0]))
        yy = (Qs.T @ b)[:rank]
        zr = scipy.linalg.solve_triangular(Rs[:rank, :rank], yy)
        z = np.zeros(rank)
        for k in range(rank - 1, -1, -1):
            acc = yy[k]
            for c in range(k + 1, rank):
                acc -= Rs[k, c] * z[c]
            z[k] = acc / Rs[k, k]
        nz += np.array_equal(z, zr)
    print(f"R {nR}/{len(S)} Q {nQ}/{len(S)} y {ny}/{len(S)} trsv {nz}/{len(S)}")


def gemv_cols(C, v, tailkind, blockcols=4):
    n = C.shape[1]
    n1 = n - n % blockcols
    out = np.zeros(n)
    for c in range(n):
        kind = "bp" if c < n1 else tailkind
        if kind in ("bp", "ap", "bf", "af"):
            out[c] = gemv_ob(C[:, c:c + 1], v, kind)[0]
        else:
            out[c] = gemv_t(C[:, c:c + 1], v, kind)[0]
    return out


if __name__ == "__main__" and "tails" in sys.argv:
    S = systems(12, 8) + systems(10, 6) + systems(9, 3)
    for tk in ("bp", "ap", "seq", "seqfma", "fma2", "fma4"):
        def apply_h2(C, v, tau, _tk=tk):
            lastv = v.size
            while lastv > 0 and v[lastv - 1] == 0.0:
                lastv -= 1
            if lastv == 0:
                return
            nz = np.nonzero(np.any(C[:lastv] != 0.0, axis=0))[0]
            lastc = int(nz[-1]) + 1 if nz.size else 0
            if lastc == 0:
                return
            w = gemv_cols(C[:lastv, :lastc], v[:lastv], _tk)
            for c in range(lastc):
                temp = -tau * w[c]
                C[:lastv, c] = [_fma(v[r], temp, C[r, c]) for r in range(lastv)]
        globals()["apply_h"] = apply_h2
        nR = 0
        for A, b in S:
            Qs, Rs, piv = scipy.linalg.qr(A, mode="economic", pivoting=True)
            n = min(A.shape)
            Af, tau, jp = factor_emul(A)
            nR += np.array_equal(np.triu(Af[:n, :]), Rs)
        print(tk, f"R exact {nR}/{len(S)}", flush=True)


if __name__ == "__main__" and "dbg" in sys.argv and "dbg2" not in sys.argv and "dbg3" not in sys.argv:
    nel, p, idx = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    A, b = systems(nel, p)[idx]
    np.set_printoptions(precision=17)
    print(A)
    _, R, piv = scipy.linalg.qr(A, mode="economic", pivoting=True)
    print("lapack", piv, np.diag(R))
    for v in [("blas", "blas", "blas"), ("cr", "blas", "blas"), ("cr", "seq", "seq")]:
        print(v, emulate(A, *v))
    print("norms blas", [blas.dnrm2(A[:, j]) for j in range(A.shape[1])])
    print("norms cr  ", [nrm2_exact_cr(A[:, j]) for j in range(A.shape[1])])


def gemv_small(C, v, variant):
    m = v.size
    m1 = m - m % 4
    out = np.zeros(C.shape[1])
    for c in range(C.shape[1]):
        col = C[:, c]
        p = [0.0] * 4
        for r in range(m1):
            p[r % 4] = _fma(col[r], v[r], p[r % 4])
        y = 0.0 + ((p[0] + p[2]) + (p[1] + p[3])) if m1 else 0.0
        lo = [(col[r], v[r]) for r in range(m1, m)]
        if lo:
            if variant == "plain":
                t = lo[0][0] * lo[0][1]
                for a, x in lo[1:]:
                    t = t + a * x
            elif variant == "fmafwd":      # fma(a_k, x_k, prev)
                t = lo[0][0] * lo[0][1]
                for a, x in lo[1:]:
                    t = _fma(a, x, t)
            elif variant == "fmafirst":    # a0*x0 + (fma chain from the right)
                t = lo[-1][0] * lo[-1][1]
                for a, x in reversed(lo[:-1]):
                    t = _fma(a, x, t)
            elif variant == "pair":        # fma(a0, x0, a1*x1) + a2*x2 ...
                t = _fma(lo[0][0], lo[0][1], lo[1][0] * lo[1][1]) if len(lo) > 1 else lo[0][0] * lo[0][1]
                for a, x in lo[2:]:
                    t = _fma(a, x, t)
            y = y + t
        out[c] = y
    return out


if __name__ == "__main__" and "dbg2" in sys.argv and "dbg3" not in sys.argv:
    S = systems(5, 1) + systems(9, 1) + systems(10, 1) + systems(9, 2) + systems(12, 8) + systems(8, 5)
    for variant in ("plain", "fmafwd", "fmafirst", "pair"):
        globals()["gemv_t"] = lambda C, v, k, _v=variant: gemv_small(C, v, _v)
        bad = 0
        for A, b in S:
            _, _, piv = scipy.linalg.qr(A, mode="economic", pivoting=True)
            r = min(A.shape)
            bad += not np.array_equal(emulate2(A, "x", "reffma")[:r], piv[:r])
        print(variant, "mismatch", bad, "of", len(S), flush=True)


if __name__ == "__main__" and "dbg3" in sys.argv:
    S = recorded_systems() + systems(5, 1) + systems(10, 1) + systems(24, 2)
    for v_small, v_big in (("fmafwd", "plain"), ("pair", "plain"), ("fmafwd", "fmafwd")):
        def g(C, v, k, _a=v_small, _b=v_big):
            return gemv_small(C, v, _a if v.size < 4 else _b)
        globals()["gemv_t"] = g
        bad = 0
        for A, b in S:
            _, _, piv = scipy.linalg.qr(A, mode="economic", pivoting=True)
            r = min(A.shape)
            bad += not np.array_equal(emulate2(A, "x", "reffma")[:r], piv[:r])
        print(v_small, v_big, "mismatch", bad, "of", len(S), flush=True)
