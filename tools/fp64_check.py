"""Checks tools/fp64_mont's products: r == a*b*b * (a*b*b)... per the chain in check_kernel."""
P = 21888242871839275222246405745257275088696311157297823662689037894645226208583
R = 1 << 288
Rinv = pow(R, -1, P)
def val(limbs):
    return sum(int(float(x)) << (48 * k) for k, x in enumerate(limbs))
bad = 0
rows = [l.split() for l in open("gpurun_out/fp64_check.txt")]
for r in rows:
    a, b, o = val(r[:6]), val(r[6:12]), val(r[12:18])
    m = lambda x, y: x * y * Rinv % P
    want = m(m(m(m(a, b), b), m(m(a, b), b)), a)
    if o % P != want % P or not (-P < o < 2 * P):
        bad += 1
print(f"{len(rows)} chains checked, {bad} mismatches")
