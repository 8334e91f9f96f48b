import sys, os, time, statistics
sys.path.insert(0, "/root/repo")
import torch
import bench
from paper_2603_10242_b200 import _native as N
from paper_2603_10242_b200.stream import PipelinedProver, pin_block
ctx = N.context(0)
n = 12800
made = [bench.canonical_block_host(n, ctx, nonce_base=k * n, slot=40 + k) for k in range(30)]
pins = [pin_block(fb, rv, rx) for fb, rv, rx in made]
for graphs in (False, True, False, True):
    pp = PipelinedProver(lanes=8, max_tx=n, max_payload=int(made[0][0].offs[n]) + 64, max_revs=1, graphs=graphs)
    for k in range(8):
        pp.submit(*made[k], pinned=pins[k])
    pp.drain()
    torch.cuda.synchronize()
    hs = []
    t0 = time.perf_counter()
    for k in range(30):
        a = time.perf_counter()
        pp.submit(*made[k], pinned=pins[k])
        hs.append((time.perf_counter() - a) * 1e6)
    res = pp.drain()
    wall = time.perf_counter() - t0
    print("graphs" if graphs else "async ", f"wall {wall*1e3:.2f} ms  {30*n/wall/1e6:.1f} M tx/s  submit median {statistics.median(hs):.0f} us  "
          f"first8 {[round(h) for h in hs[:8]]}  lat p50 {statistics.median(r.latency_ms for r in res):.3f}")
    pp.close()
