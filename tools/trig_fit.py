"""Minimax coefficients of the sin/cos polynomials in csrc/rb_trig.cuh.

After reduction by pi, |r| <= pi/2 and z = r^2:
    cos r = 1 + z Q(z)        sin r = r + r z S(z)
Q and S minimise the absolute error of the whole expression (weighted Remez
exchange in 50-digit mpmath).  Prints the coefficients (lowest order first)
and the minimax error for the degrees used: double Q7 / S7 (general), Q6
(Weierstrass), float Q4 / S3.
    python tools/trig_fit.py
"""
import mpmath as mp

mp.mp.dps = 50
R2 = (mp.pi / 2) ** 2
EPS = mp.mpf("1e-30")


def remez_weighted(f, w, a, b, deg, iters=15):
    """Minimise max |w(x) (P(x) - f(x))| over [a, b], P of degree deg."""
    n = deg + 2
    xs = [(a + b) / 2 - (b - a) / 2 * mp.cos(mp.pi * i / (n - 1)) for i in range(n)]
    err_max = None
    for _ in range(iters):
        A = mp.matrix([[x ** j * w(x) for j in range(deg + 1)] + [(-1) ** i] for i, x in enumerate(xs)])
        y = mp.matrix([f(x) * w(x) for x in xs])
        sol = mp.lu_solve(A, y)
        c = [sol[j] for j in range(deg + 1)]
        grid = [a + (b - a) * i / 4000 for i in range(4001)]
        ev = [(mp.polyval(c[::-1], x) - f(x)) * w(x) for x in grid]
        err_max = max(abs(e) for e in ev)
        ext = [grid[0]] + [grid[i] for i in range(1, 4000)
                           if (ev[i] - ev[i - 1]) * (ev[i + 1] - ev[i]) <= 0] + [grid[-1]]
        if len(ext) != n:
            break
        xs = ext
    return c, err_max


def cos_q(z):
    return (mp.cos(mp.sqrt(z)) - 1) / z if z > EPS else mp.mpf(-0.5)


def sin_s(z):
    return (mp.sin(mp.sqrt(z)) - mp.sqrt(z)) / (z * mp.sqrt(z)) if z > EPS else mp.mpf(-1) / 6


def main():
    for name, f, w, deg in (("cos Q (double)", cos_q, lambda z: max(z, EPS), 7),
                            ("cos Q (Weierstrass)", cos_q, lambda z: max(z, EPS), 6),
                            ("sin S (double)", sin_s, lambda z: max(z * mp.sqrt(z), EPS), 7),
                            ("cos Q (float)", cos_q, lambda z: max(z, EPS), 4),
                            ("sin S (float)", sin_s, lambda z: max(z * mp.sqrt(z), EPS), 3)):
        c, err = remez_weighted(f, w, mp.mpf(0), R2, deg)
        print(f"{name}, degree {deg}: max abs error {float(err):.3g}")
        print("   ", [repr(float(x)) for x in c])


if __name__ == "__main__":
    main()
