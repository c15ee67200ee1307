"""Provenance of the log1p polynomial in k_mlp_tc_sp.cu (K2s): a degree-9 Chebyshev fit of
log1p(t) on [0, 1], converted to monomial coefficients and rounded to fp32; prints the
coefficients and the max error of fp32 Horner evaluation (kernel constants, not part of the
oracle).  python tools/fit_log1p.py"""
import numpy as np

t = np.linspace(0, 1, 400001)
y = np.log1p(t)
c = np.polynomial.chebyshev.Chebyshev.fit(t, y, 9, domain=[0, 1])
p = c.convert(kind=np.polynomial.Polynomial, domain=[0, 1], window=[0, 1]).coef.astype(np.float32)
acc = np.full(t.shape, p[-1], np.float32)
for k in range(len(p) - 2, -1, -1):
    acc = (acc * t.astype(np.float32) + p[k]).astype(np.float32)
print("coefficients (c0..c9):", ", ".join("%.9ef" % v for v in p))
print("max |poly - log1p| in fp32 Horner on [0, 1]: %.3e" % np.abs(acc - y).max())
