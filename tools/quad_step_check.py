"""Offline check of the trapezoid step of the Gamma-mixture quadrature (matern_rho.cuh):
the discretisation error of ln ρ at h = min(0.165, α σ), summed in 30-digit arithmetic
(mpmath) so that only the step and the e^-40 cut count, against mpmath besselk, for
κ ∈ [0.02, 500] and s over 2^-40 .. 2^17.  Prints the worst |Δ ln ρ| / max(1, |ln ρ|) per α.
Measured on this grid: α = 0.45: 1.9e-17, α = 0.6: 1.3e-16, α = 0.7: 3.6e-16; a denser
grid around κ r ≈ 13 (where 0.6 σ meets the 0.165 cap) gives 1.0e-15 for α = 0.6 at
κ = 13, s = 12.9 — so the kernel keeps α = 0.45.  usage: python tools/quad_step_check.py"""
import mpmath as mp
mp.mp.dps = 30
def logrho_ref(k, s):
    z = mp.sqrt(s)
    return (1-k)*mp.log(2) - mp.loggamma(k) + k*mp.log(z) + mp.log(mp.besselk(k, z))
def trap(k, s, alpha, hmax=0.165, cut=40):
    k = mp.mpf(k); s = mp.mpf(s)
    q = s/(k*k); r = mp.sqrt(1+q); xs = mp.log((1+r)/2)
    h = min(mp.mpf(hmax), alpha/mp.sqrt(k*r))
    a = s/(4*k)
    G = lambda x: k*(x - (mp.e**x - 1)) - a*mp.e**(-x)
    gs = G(xs)
    tot = mp.mpf(1)
    for sgn in (1, -1):
        i = 1
        while True:
            g = G(xs + sgn*i*h) - gs
            if g < -cut: break
            tot += mp.e**g; i += 1
    lnC = k*mp.log(k) - k - mp.loggamma(k)
    return lnC + gs + mp.log(h*tot)
worst = {}
for alpha in (0.45, 0.6, 0.7):
    w = 0
    for k in (0.02, 0.1, 0.5, 2.0, 10.0, 100.0, 500.0):
        for e in (-40, -20, -8, -2, 0, 2, 5, 8, 11, 14, 17):
            s = mp.mpf(2)**e * mp.mpf(1.37)
            ref = logrho_ref(k, s)
            if ref < -745: continue
            err = abs(trap(k, s, alpha) - ref) / max(1, abs(ref))
            w = max(w, float(err))
    print(alpha, w)
