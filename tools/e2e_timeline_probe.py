"""GPU timeline of the chunked host-buffer Ax pipeline (copy-engine H2D of u
chunk c || Ax chunk c || copy-engine D2H of w chunk c): every op bracketed
by CUDA events, all ops queued behind a sleep gate first so host enqueue
time is not on the timeline.  Prints per-chunk start/end (us from the gate)
and the total, for a few chunk sizes; also a variant with w written by the
kernel into mapped host memory (no D2H)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2005_13425_b200 as sb  # noqa: E402
from paper_2005_13425_b200._lib import load  # noqa: E402
from paper_2005_13425_b200.kernels import _basis_host_ptrs  # noqa: E402

E, n = 4096, 10
per = n ** 3
b = sb.build_basis(n)
lib = load()
pdx, pdxt = _basis_host_ptrs(b)
u_d = sb.random_field(E, n, 1, device="cuda")
g_d = sb.random_field(6 * E, n, 2, device="cuda").reshape(E, 6, n, n, n)
u_h = u_d.cpu().pin_memory()
w_h = torch.empty(u_h.shape, dtype=torch.float64).pin_memory()
ud, wd = torch.empty_like(u_d), torch.empty_like(u_d)
main = torch.cuda.current_stream()
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()


def ev():
    e = torch.cuda.Event(enable_timing=True)
    return e


def run_h2d_first(chunk_el, variant=0):
    """Submission order B: every H2D chunk queued first, then per chunk the
    kernel and its D2H."""
    gate = ev()
    torch.cuda._sleep(int(3e6))
    gate.record(main)
    s_in.wait_event(gate)
    s_out.wait_event(gate)
    rows = []
    spans = list(range(0, E, chunk_el))
    for e0 in spans:
        e1 = min(E, e0 + chunk_el)
        r = {k: ev() for k in ("h0", "h1", "k0", "k1", "d0", "d1")}
        with torch.cuda.stream(s_in):
            r["h0"].record(s_in)
            ud[e0:e1].copy_(u_h[e0:e1], non_blocking=True)
            r["h1"].record(s_in)
        rows.append(r)
    for e0, r in zip(spans, rows):
        e1 = min(E, e0 + chunk_el)
        main.wait_event(r["h1"])
        r["k0"].record(main)
        rc = lib.sem_ax_variant(ud[e0:e1].data_ptr(), g_d[e0:e1].data_ptr(), pdx, pdxt,
                                wd[e0:e1].data_ptr(), e1 - e0, n, variant, main.cuda_stream)
        assert rc == 0, lib.sem_last_error()
        r["k1"].record(main)
        with torch.cuda.stream(s_out):
            s_out.wait_event(r["k1"])
            r["d0"].record(s_out)
            w_h[e0:e1].copy_(wd[e0:e1], non_blocking=True)
            r["d1"].record(s_out)
    end = ev()
    main.wait_stream(s_out)
    end.record(main)
    torch.cuda.synchronize()
    t = lambda e: round(gate.elapsed_time(e) * 1e3, 1)  # noqa: E731
    return t(end), [{"h": (t(r["h0"]), t(r["h1"])), "k": (t(r["k0"]), t(r["k1"])),
                     "d": (t(r["d0"]), t(r["d1"]))} for r in rows]


def run(chunk_el, mapped_w=False, variant=0):
    gate = ev()
    torch.cuda._sleep(int(3e6))
    gate.record(main)
    s_in.wait_event(gate)
    s_out.wait_event(gate)
    rows = []
    wmap = w_h  # torch pinned tensors are mapped (UVA): the kernel can store to them
    for e0 in range(0, E, chunk_el):
        e1 = min(E, e0 + chunk_el)
        r = {k: ev() for k in ("h0", "h1", "k0", "k1", "d0", "d1")}
        with torch.cuda.stream(s_in):
            r["h0"].record(s_in)
            ud[e0:e1].copy_(u_h[e0:e1], non_blocking=True)
            r["h1"].record(s_in)
        main.wait_event(r["h1"])
        r["k0"].record(main)
        out = wmap[e0:e1] if mapped_w else wd[e0:e1]
        rc = lib.sem_ax_variant(ud[e0:e1].data_ptr(), g_d[e0:e1].data_ptr(), pdx, pdxt,
                                out.data_ptr(), e1 - e0, n, variant, main.cuda_stream)
        assert rc == 0, lib.sem_last_error()
        r["k1"].record(main)
        if not mapped_w:
            with torch.cuda.stream(s_out):
                s_out.wait_event(r["k1"])
                r["d0"].record(s_out)
                w_h[e0:e1].copy_(wd[e0:e1], non_blocking=True)
                r["d1"].record(s_out)
        rows.append(r)
    end = ev()
    main.wait_stream(s_out)
    end.record(main)
    torch.cuda.synchronize()
    t = lambda e: round(gate.elapsed_time(e) * 1e3, 1)  # noqa: E731
    out = []
    for r in rows:
        d = {"h": (t(r["h0"]), t(r["h1"])), "k": (t(r["k0"]), t(r["k1"]))}
        if not mapped_w:
            d["d"] = (t(r["d0"]), t(r["d1"]))
        out.append(d)
    return t(end), out


for mb in (8, 4, 2):
    ce = max(1, int(mb * 2 ** 20 // (8 * per)))
    best = min((run_h2d_first(ce) for _ in range(3)), key=lambda x: x[0])
    print(json.dumps({"chunk_MB": mb, "order": "h2d_first", "total_us": best[0], "chunks": best[1]}),
          flush=True)
for mb, mapped, var in ((8, False, 0), (4, False, 0), (4, True, 63)):
    ce = max(1, int(mb * 2 ** 20 // (8 * per)))
    best = None
    for _ in range(3):
        tot, rows = run(ce, mapped, var)
        if best is None or tot < best[0]:
            best = (tot, rows)
    ok = torch.equal(w_h.cuda(), torch.empty_like(u_d)) if False else None
    print(json.dumps({"chunk_MB": mb, "order": "interleaved", "mapped_w": mapped, "total_us": best[0],
                      "chunks": best[1]}), flush=True)
