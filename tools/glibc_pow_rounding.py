# Measures how often glibc pow(u, b) (u in (0,1), b in [0,4), the mini-render
# draws) differs from the correctly rounded value (50-digit Decimal).
# Result in this image: 22 of 20000 (0.11%) -> no independent pow can be
# bit-identical to the reference; DESIGN.md section 5.
import numpy as np, math, ctypes
from decimal import Decimal, getcontext
getcontext().prec = 50
libm = ctypes.CDLL("libm.so.6"); libm.pow.restype=ctypes.c_double; libm.pow.argtypes=[ctypes.c_double]*2
rs=np.random.RandomState(1)
N=20000
bad=0
for i in range(N):
    u=float(rs.randint(1,2**53))*2.0**-53
    b=4.0*float(rs.randint(0,2**53))*2.0**-53
    g=libm.pow(u,b)
    exact=(Decimal(b)*Decimal(u).ln()).exp()
    # correctly rounded double of exact
    cr=float(exact)   # Decimal->float conversion is correctly rounded
    if cr!=g: bad+=1
print("glibc pow != correctly rounded:", bad, "of", N)
