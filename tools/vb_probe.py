"""Variable-base MSM throughput at block-key sizes (G1 2^22..2^26, G2 2^24):
2^20 generated bases tiled on the device, random scalars; CUDA events."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_10242_b200 import _native as N  # noqa: E402

ctx = N.context(0)
R = 0x30644E72E131A029B85045B68181585D2833E84879B9709143E1F593F0000001


G2 = [10857046999023057135944570762232829481370756359578518086990519993285655852781,
      11559732032986387107991004021392285783925812861821192530917403151452391805634,
      8495653923123431417604973247489272438418190587263600148770280649306958101930,
      4082367875863433681332203403145435568316851327593401208105741076214120093531]


def gen(group, n0=1 << 20):
    rng = np.random.default_rng(group)
    k = rng.integers(0, 2**63, size=(n0, 4), dtype=np.uint64)
    k[:, 3] &= (1 << 61) - 1
    if group == 1:
        G = np.frombuffer((1).to_bytes(32, "little") + (2).to_bytes(32, "little"), np.uint8).copy()
    else:
        G = np.frombuffer(b"".join(v.to_bytes(32, "little") for v in G2), np.uint8).copy()
    pts = np.zeros(64 * group * n0, np.uint8)
    ctx.call("acegpu_bn_scalar_muls", group, G, k.view(np.uint8).reshape(-1), n0, pts)
    return torch.from_numpy(pts).cuda()


def check_vs_fixed(group, logn, base):
    """VB == fixed base (window tables) at the same size."""
    n = 1 << logn
    reps = n // (base.numel() // (64 * group))
    pts = base.repeat(reps)
    sc = torch.randint(0, 256, (n, 32), dtype=torch.uint8, device="cuda")
    sc[:, 31] &= 0x1F
    outs = []
    for vb in (1, 0):
        h = C.c_void_p()
        if vb:
            ctx.call("acegpu_bn_msm_prepare_vb", group, pts.data_ptr(), n, 1, 0, C.byref(h))
        else:
            ctx.call("acegpu_bn_msm_prepare", group, pts.data_ptr(), n, 1, C.byref(h))
        out = torch.empty(64 * group, dtype=torch.uint8, device="cuda")
        s = torch.cuda.current_stream()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(2):
            a.record(s)
            ctx.call("acegpu_bn_msm_run_dev", s.cuda_stream, h, sc.data_ptr(), out.data_ptr())
            b.record(s)
            torch.cuda.synchronize()
        print(f"G{group} 2^{logn} {'vb' if vb else 'fixed'}: {a.elapsed_time(b):.1f} ms", flush=True)
        outs.append(out.cpu().numpy().tobytes())
        N.lib().acegpu_bn_msm_free(h)
        torch.cuda.empty_cache()
    print("vb == fixed:", outs[0] == outs[1], flush=True)
    assert outs[0] == outs[1]


def run(group, logn, base):
    n = 1 << logn
    reps = n // (base.numel() // (64 * group))
    pts = base.repeat(reps)
    sc = torch.randint(0, 256, (n, 32), dtype=torch.uint8, device="cuda")
    sc[:, 31] &= 0x1F
    h = C.c_void_p()
    ctx.call("acegpu_bn_msm_prepare_vb", group, pts.data_ptr(), n, 1, 0, C.byref(h))
    del pts
    out = torch.empty(64 * group, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    ts, res = [], []
    for r in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        ctx.call("acegpu_bn_msm_run_dev", s.cuda_stream, h, sc.data_ptr(), out.data_ptr())
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
        res.append(out.cpu().numpy().tobytes())
    N.lib().acegpu_bn_msm_free(h)
    print("  times", [round(t, 1) for t in ts], "same result", len(set(res)) == 1)
    W = (255 + 19) // 20  # the variable-base windows (c = 20)
    print(f"G{group} vb 2^{logn}: {min(ts):.1f} ms ({n * W / min(ts) / 1e6:.2f} G entries/s)", flush=True)
    del sc
    torch.cuda.empty_cache()


if __name__ == "__main__":
    b1 = gen(1)
    if '--check' in sys.argv:
        check_vs_fixed(1, 26, b1)
    for L in (20, 22, 24, 26):
        run(1, L, b1)
    del b1
    b2 = gen(2, 1 << 18)
    for L in (20, 24):
        run(2, L, b2)
