"""Pinned host -> device copy bandwidth (the e2e floor): whole vs chunked,
one vs two streams. Not a benchmark."""
import torch

MB = 1 << 20


def timed(fn, reps=30):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


for size in (4, 16, 27, 64):
    n = size * MB
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h.fill_(1)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    st = [torch.cuda.Stream() for _ in range(2)]

    def whole():
        d.copy_(h, non_blocking=True)

    def chunked(k=2 * MB, streams=1):
        cur = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(cur)
        for i, o in enumerate(range(0, n, k)):
            ss = st[i % streams]
            ss.wait_event(ev)
            with torch.cuda.stream(ss):
                d[o:o + k].copy_(h[o:o + k], non_blocking=True)
        for ss in st[:streams]:
            e2 = torch.cuda.Event()
            e2.record(ss)
            cur.wait_event(e2)

    for name, fn in (("whole", whole), ("chunk2M", chunked),
                     ("chunk2M x2 streams", lambda: chunked(streams=2)),
                     ("chunk8M x2 streams", lambda: chunked(8 * MB, 2))):
        ms = timed(fn)
        print(f"{size:3d} MiB {name:20s} {ms:.3f} ms {n / ms / 1e6:.1f} GB/s")
    ms = timed(lambda: h.copy_(d, non_blocking=True))
    print(f"{size:3d} MiB {'D2H':20s} {ms:.3f} ms {n / ms / 1e6:.1f} GB/s")
