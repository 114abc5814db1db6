"""Generates the Taylor coefficients of 1/Γ(1+μ) = Σ_{k≥0} a_k μ^k (A&S 6.1.34
shifted by one) used by the device Temme series constants gam1, gam2 of the
fractional Bessel order μ ∈ [−1/2, 1/2].  Run once; output pasted into
bessel_k.cuh.  mpmath at 60 digits (an independent library, not the oracle)."""
import mpmath

mpmath.mp.dps = 60
a = mpmath.taylor(lambda z: mpmath.rgamma(1 + z), 0, 29)
for k, v in enumerate(a):
    print(f"    {mpmath.nstr(v, 22)},  // a_{k}")
