"""Prints the (hi, lo) double-double table of atan(k/64), k = 0..64, and the
pi, pi/2 splits used by paper_2008_00409_b200/csrc/cr_atan2.cuh (mpmath at
200 bits; hex literals so the values parse exactly)."""
import mpmath as mp

mp.mp.prec = 200


def dd(v):
    hi = float(v)
    return hi, float(v - mp.mpf(hi))


for k in range(65):
    hi, lo = dd(mp.atan(mp.mpf(k) / 64))
    print(f"    {hi.hex()}, {lo.hex()},")
for name, v in (("pi", mp.pi), ("pi/2", mp.pi / 2)):
    hi, lo = dd(v)
    print(f"// {name}: {hi.hex()} {lo.hex()}")
