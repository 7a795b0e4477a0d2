"""Constants of csrc/fastmath.cuh: 2^(j/64) for j = 0..63 correctly rounded to
fp64 (80-digit decimal arithmetic, then one rounding), and ln2/64 split into a
36-significant-bit head (kd * head exact for |kd| < 2^17) and its tail."""
import math
from decimal import Decimal, getcontext

getcontext().prec = 80
ln2 = Decimal(2).ln()
for j in range(64):
    print(f"    {float((Decimal(j) / 64 * ln2).exp()).hex()},")
l = ln2 / 64
m, e = math.frexp(float(l))
hi = math.ldexp(round(m * 2 ** 36), e - 36)
print("ln2/64 head", hi.hex(), "tail", float(l - Decimal(hi)).hex(), "64/ln2", float(Decimal(64) / ln2).hex())
