"""Copy-engine behaviour behind the host-buffer Ax: 32.8 MB H2D and D2H
(pinned), whole and in chunks, alone and concurrently on two streams, and
the kernel's own zero-copy read / write rates.  CUDA-event timed."""
import json
import torch

MB = 2 ** 20
total = 32768000
h_in = torch.empty(total // 8, dtype=torch.float64).pin_memory()
h_out = torch.empty(total // 8, dtype=torch.float64).pin_memory()
d_in = torch.empty(total // 8, dtype=torch.float64, device="cuda")
d_out = torch.ones(total // 8, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def chunks(cb):
    per = cb // 8
    return [(i, min(i + per, total // 8)) for i in range(0, total // 8, per)]


def h2d(cb, stream=None):
    st = stream or torch.cuda.current_stream()
    with torch.cuda.stream(st):
        for a, b in chunks(cb):
            d_in[a:b].copy_(h_in[a:b], non_blocking=True)


def d2h(cb, stream=None):
    st = stream or torch.cuda.current_stream()
    with torch.cuda.stream(st):
        for a, b in chunks(cb):
            h_out[a:b].copy_(d_out[a:b], non_blocking=True)


def both(cb):
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    h2d(cb, s1)
    d2h(cb, s2)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


for mb in (32, 8, 4, 2, 1, 0.5):
    cb = int(mb * MB)
    r = {"chunk_MB": mb, "h2d_ms": timed(lambda: h2d(cb)), "d2h_ms": timed(lambda: d2h(cb)),
         "duplex_ms": timed(lambda: both(cb))}
    r["h2d_GBs"] = total / r["h2d_ms"] / 1e6
    r["d2h_GBs"] = total / r["d2h_ms"] / 1e6
    r["duplex_GBs_total"] = 2 * total / r["duplex_ms"] / 1e6
    print(json.dumps({k: round(v, 4) if isinstance(v, float) else v for k, v in r.items()}), flush=True)
