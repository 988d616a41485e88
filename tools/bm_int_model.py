# Python integer model of the integer Box-Muller transform (philox_bm.cuh box_muller_int),
# exact integer arithmetic, checked against 60-digit mpmath references (max error 3e-16 max(1,|z|)).
# Python integer model of the integer Box-Muller transform (exact integer arithmetic),
# validated against mpmath.  Mirrors the planned CUDA code op by op.
import mpmath as mp
import random
mp.mp.dps = 60
M64 = (1 << 64) - 1

def umulhi(a, b):
    return (a * b) >> 64

def smulhi(a, b):  # signed 64x64 -> high 64 (floor)
    return (a * b) >> 64

# ---------------- tables
PI = mp.pi
K_B = int(mp.nint((PI / 2) * 2 ** 63))           # bq = umulhi(dm << 14, K_B)
SIN63 = [int(mp.nint(mp.sin((PI / 2) * j / 64) * 2 ** 63)) for j in range(64)]
COS63 = [int(mp.nint(mp.cos((PI / 2) * j / 64) * 2 ** 63)) for j in range(64)]
S3, S5, S7 = [int(mp.nint(2 ** 64 / mp.factorial(k))) for k in (3, 5, 7)]
C2, C4, C6, C8 = [int(mp.nint(2 ** 64 / mp.factorial(k))) for k in (2, 4, 6, 8)]

# invc: 9-significant-bit approximation of 1/(1 + (i + 1/2)/128); invc[127] = 1/2
CI = []
for i in range(128):
    if i == 127:
        CI.append(256)        # 1/2 = 256 / 512
    else:
        v = 1 / (1 + (i + 0.5) / 128)
        CI.append(int(round(v * 512)))
TWO_LN2_Q57 = int(mp.nint(2 * mp.log(2) * 2 ** 57))
LNINV = [int(mp.nint(2 * mp.log(mp.mpf(c) / 512) * 2 ** 57)) for c in CI]
LNINV[127] = -TWO_LN2_Q57
# P(r) = log1p(r)/r = sum_{k>=0} (-r)^k/(k+1), Q62 coefficients, r in Q61
PK = [int(mp.nint(mp.mpf(1) / (k + 1) * 2 ** 62)) for k in range(10)]

def to_double_u(v, scale):   # unsigned integer v * 2^-scale -> nearest double (ties even)
    if v == 0:
        return 0.0
    return float(mp.mpf(v) * mp.mpf(2) ** -scale)   # model: correctly rounded

def sincos(n2):
    k = n2 >> 51
    j = (n2 >> 45) & 63
    dm = n2 & ((1 << 45) - 1)
    bq = umulhi(dm << 14, K_B)                 # Q64
    b2 = umulhi(bq, bq)                        # Q64
    t = S5 - umulhi(b2, S7)
    t = S3 - umulhi(b2, t)
    t = umulhi(b2, t)                          # b^2 (1/6 - b^2 (...))  Q64
    sinb = bq - umulhi(bq, t)                  # Q64
    u = C6 - umulhi(b2, C8)
    u = C4 - umulhi(b2, u)
    u = C2 - umulhi(b2, u)
    u = umulhi(b2, u)                          # b^2 (1/2 - ...)  Q64
    cb = (1 << 63) - (u >> 1)                  # Q63
    sb = sinb >> 1                             # Q63
    sa, ca = SIN63[j], COS63[j]
    mul63 = lambda a, b: (a * b) >> 63
    S = mul63(sa, cb) + mul63(ca, sb)
    C = mul63(ca, cb) - mul63(sa, sb)
    s_, c_ = to_double_u(S, 63), to_double_u(C, 63)
    if k == 0: return s_, c_
    if k == 1: return c_, -s_
    if k == 2: return -s_, -c_
    return -c_, s_

def m2ln(n1):
    if n1 == 1 << 53:
        return 0.0
    e = n1.bit_length() - 1
    mant = (n1 << (52 - e)) & ((1 << 52) - 1)
    i = mant >> 45
    P = ((1 << 52) + mant) * CI[i]             # m * invc * 2^61, exact
    R = P - (1 << 61)                          # r in Q61, exact, |R| < 2^54
    # P(r) in Q62 by Horner: p = PK[8]; p = PK[k] - r p ...
    p = PK[8]
    for kk in range(7, -1, -1):
        p = PK[kk] - smulhi(R << 3, p)         # (R<<3) is r in Q64; smulhi(Q64, Q62) -> Q62
    B128 = -2 * R * p                          # -2 r P(r) in Q(61+62) = Q123, exact product
    A = (53 - e) * TWO_LN2_Q57 + LNINV[i]      # Q57, >= 0
    Bd = float(mp.mpf(B128) * mp.mpf(2) ** -123)
    Ad = to_double_u(A, 57)
    return Ad + Bd

def bm(w0, w1):
    n1 = (w0 >> 11) + 1
    n2 = w1 >> 11
    x = m2ln(n1)
    rho = float(mp.sqrt(mp.mpf(x)))            # model: correctly rounded sqrt
    sn, cs = sincos(n2)
    return rho * cs, rho * sn

def ref(w0, w1):
    u1 = mp.mpf((w0 >> 11) + 1) * mp.mpf(2) ** -53
    u2 = mp.mpf(w1 >> 11) * mp.mpf(2) ** -53
    rho = mp.sqrt(-2 * mp.log(u1))
    return rho * mp.cos(2 * mp.pi * u2), rho * mp.sin(2 * mp.pi * u2)

random.seed(1)
words = [(random.getrandbits(64), random.getrandbits(64)) for _ in range(3000)]
# edge cases: u1 -> 1, u1 -> 0, quadrant boundaries
for t in range(60):
    words.append(((1 << 64) - 1 - random.getrandbits(min(t + 1, 63)), random.getrandbits(64)))
    words.append((random.getrandbits(t + 1), random.getrandbits(64)))
for quad in range(4):
    for j in (0, 1, 31, 63):
        for d in (0, 1, 2 ** 11, -(2 ** 11)):
            n2 = (quad << 51) + (j << 45)
            words.append((random.getrandbits(64), ((n2 << 11) + d) % (1 << 64)))
words += [(0, 0), ((1 << 64) - 1, (1 << 64) - 1)]
worst = 0
for w0, w1 in words:
    z = bm(w0, w1)
    r = ref(w0, w1)
    for a, b in zip(z, r):
        err = abs(mp.mpf(a) - b) / max(1, abs(b))
        worst = max(worst, float(err))
print("max err / max(1,|z|):", worst)
