import mpmath as mp, numpy as np
mp.mp.dps = 50
def fit(f, a, b, deg):
    # Chebyshev interpolation (near-minimax) of f on [a,b] in z, then monomial coeffs
    n = deg + 1
    nodes = [ (a+b)/2 + (b-a)/2*mp.cos(mp.pi*(2*i+1)/(2*n)) for i in range(n)]
    # solve Vandermonde in high precision
    A = mp.matrix([[x**j for j in range(n)] for x in nodes])
    y = mp.matrix([f(x) for x in nodes])
    c = mp.lu_solve(A, y)
    return [c[j] for j in range(n)]
def remez(f, a, b, deg, iters=12):
    n = deg + 2
    xs = [ (a+b)/2 - (b-a)/2*mp.cos(mp.pi*i/(n-1)) for i in range(n)]
    for it in range(iters):
        A = mp.matrix([[x**j for j in range(deg+1)] + [(-1)**i] for i, x in enumerate(xs)])
        y = mp.matrix([f(x) for x in xs])
        sol = mp.lu_solve(A, y)
        c = [sol[j] for j in range(deg+1)]
        E = sol[deg+1]
        err = lambda x: mp.polyval(c[::-1], x) - f(x)
        # find extrema on a fine grid
        grid = [a + (b-a)*i/4000 for i in range(4001)]
        ev = [err(x) for x in grid]
        ext = [grid[0]]
        for i in range(1, 4000):
            if (ev[i]-ev[i-1])*(ev[i+1]-ev[i]) <= 0: ext.append(grid[i])
        ext.append(grid[-1])
        if len(ext) != n:
            break
        xs = ext
    return c, E
import sys
R = mp.pi/2
f = lambda z: mp.cos(mp.sqrt(z))
for deg in (8, 9, 10):
    c, E = remez(f, mp.mpf(0), R**2, deg)
    cd = [float(x) for x in c]
    # evaluate in double Horner with fma emulation via mpmath rounding
    rs = np.linspace(-1.5707963267948966, 1.5707963267948966, 20001)
    worst = 0
    for r in rs[::7]:
        z = float(mp.mpf(r)*mp.mpf(r))
        p = cd[-1]
        for k in range(len(cd)-2, -1, -1):
            p = float(mp.mpf(p)*mp.mpf(z) + mp.mpf(cd[k]))  # fma
        worst = max(worst, abs(p - float(mp.cos(mp.mpf(r)))))
    print(deg, float(E), worst, [repr(x) for x in cd])
