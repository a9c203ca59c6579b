"""PCIe copy granularity probe for the host-buffer (e2e) pipeline -- dev tool.

Times the C1 step's bytes (H2D 168 MB: q 134 MB + k 16.8 + v 16.8; D2H 134 MB) as
  a) one H2D copy / one D2H copy, alone and concurrently (two streams),
  b) the pipeline's copy granularity: 27 H2D copies (k/v halves, query rows, 22 q chunks)
     and 22 D2H chunk copies, with an event after every copy, alone and concurrently.
If (b) is as fast as (a), copy granularity is not what separates e2e from its copy floor.
"""
import torch

MB = 1 << 20
q_b, kv_b, o_b = 134217728, 16777216, 134217728
dev = torch.device("cuda:0")
hq = torch.empty(q_b, dtype=torch.uint8).pin_memory()
hk = torch.empty(2 * kv_b, dtype=torch.uint8).pin_memory()
ho = torch.empty(o_b, dtype=torch.uint8).pin_memory()
dq = torch.empty(q_b, dtype=torch.uint8, device=dev)
dk = torch.empty(2 * kv_b, dtype=torch.uint8, device=dev)
do = torch.empty(o_b, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
frac = [0, 1, 2, 4, 6, 8, 12, 16, 20, 24, 28, 32]


def chunks(total, n_blocks=2):
    per = total // n_blocks
    out = []
    for b in range(n_blocks):
        for c in range(len(frac) - 1):
            a, e = per * frac[c] // 32, per * frac[c + 1] // 32
            out.append((b * per + a, b * per + e))
    return out


EVENTS = [True]


def h2d(fine):
    with torch.cuda.stream(s1):
        if not fine:
            dq.copy_(hq, non_blocking=True)
            dk.copy_(hk, non_blocking=True)
            return
        half = kv_b // 2
        for a, e in ((0, half), (kv_b, kv_b + half), (half, kv_b), (kv_b + half, 2 * kv_b)):
            dk[a:e].copy_(hk[a:e], non_blocking=True)
            if EVENTS[0]:
                torch.cuda.current_stream().record_event()
        for a, e in chunks(q_b):
            dq[a:e].copy_(hq[a:e], non_blocking=True)
            if EVENTS[0]:
                torch.cuda.current_stream().record_event()


def d2h(fine):
    with torch.cuda.stream(s2):
        if not fine:
            ho.copy_(do, non_blocking=True)
            return
        for a, e in chunks(o_b):
            ho[a:e].copy_(do[a:e], non_blocking=True)
            if EVENTS[0]:
                torch.cuda.current_stream().record_event()


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s1.wait_stream(torch.cuda.current_stream())
        s2.wait_stream(torch.cuda.current_stream())
        fn()
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for fine in (False, True):
    tag = "27/22 copies" if fine else "1 copy each "
    a = timed(lambda: h2d(fine))
    b = timed(lambda: d2h(fine))
    c = timed(lambda: (h2d(fine), d2h(fine)))
    print(f"{tag}: H2D 168MB {a:.3f} ms ({(q_b + 2 * kv_b) / a / 1e6:.1f} GB/s)  D2H 134MB {b:.3f} ms  "
          f"both {c:.3f} ms ({(q_b + 2 * kv_b + o_b) / c / 1e6:.1f} GB/s)")
print(f"fine H2D + 1 D2H copy : both {timed(lambda: (h2d(True), d2h(False))):.3f} ms")
print(f"1 H2D copy + fine D2H : both {timed(lambda: (h2d(False), d2h(True))):.3f} ms")


def even(total, n):
    return [(total * i // n, total * (i + 1) // n) for i in range(n)]


def h2d_n(n, ev=False):
    with torch.cuda.stream(s1):
        dk.copy_(hk, non_blocking=True)
        for a, e in even(q_b, n):
            dq[a:e].copy_(hq[a:e], non_blocking=True)
            if ev:
                torch.cuda.current_stream().record_event()


def d2h_n(n, ev=False):
    with torch.cuda.stream(s2):
        for a, e in even(o_b, n):
            ho[a:e].copy_(do[a:e], non_blocking=True)
            if ev:
                torch.cuda.current_stream().record_event()


for n in (2, 4, 8, 16, 32):
    print(f"even chunks n={n:2d}: both {timed(lambda: (h2d_n(n), d2h_n(n))):.3f} ms   "
          f"H2D n, D2H 1: {timed(lambda: (h2d_n(n), d2h_n(1))):.3f}   H2D 1, D2H n: {timed(lambda: (h2d_n(1), d2h_n(n))):.3f}")

EVENTS[0] = False
print(f"27/22 uneven copies, no events: both {timed(lambda: (h2d(True), d2h(True))):.3f} ms")
EVENTS[0] = True
print(f"even 22/22 with events: both {timed(lambda: (h2d_n(22, True), d2h_n(22, True))):.3f} ms; "
      f"even 22/22 no events {timed(lambda: (h2d_n(22), d2h_n(22))):.3f}")
for n in (11, 22, 44):
    print(f"even {n}/{n} with events: {timed(lambda: (h2d_n(n, True), d2h_n(n, True))):.3f} ms; H2D {n} + D2H 8: "
          f"{timed(lambda: (h2d_n(n, True), d2h_n(8, True))):.3f}; H2D {n} + D2H 44: {timed(lambda: (h2d_n(n, True), d2h_n(44, True))):.3f}")


def aligned(total, n, al):
    b = [min(total, (total * i // n + al // 2) // al * al) for i in range(n + 1)]
    b[-1] = total
    return [(b[i], b[i + 1]) for i in range(n) if b[i + 1] > b[i]]


def both_al(n, al, nd=None):
    def f():
        with torch.cuda.stream(s1):
            dk.copy_(hk, non_blocking=True)
            for a, e in aligned(q_b, n, al):
                dq[a:e].copy_(hq[a:e], non_blocking=True)
                torch.cuda.current_stream().record_event()
        with torch.cuda.stream(s2):
            for a, e in aligned(o_b, nd or n, al):
                ho[a:e].copy_(do[a:e], non_blocking=True)
                torch.cuda.current_stream().record_event()
    return timed(f)


for n in (11, 22, 32):
    print(f"n={n}: " + "  ".join(f"align {al >> 10}K {both_al(n, al):.3f}" for al in (4096, 65536, 1 << 20, 2 << 20, 4 << 20)))


s3 = torch.cuda.Stream()


def h2d_two(fine_d2h=True):
    """the pipeline's 27 H2D copies alternating over two streams (two copies in flight)"""
    def f():
        ss = [s1, s3]
        s3.wait_stream(s1)
        half = kv_b // 2
        parts = [("k", a, e) for a, e in ((0, half), (kv_b, kv_b + half), (half, kv_b), (kv_b + half, 2 * kv_b))]
        parts += [("q", a, e) for a, e in chunks(q_b)]
        for t, (w, a, e) in enumerate(parts):
            with torch.cuda.stream(ss[t % 2]):
                (dk if w == "k" else dq)[a:e].copy_((hk if w == "k" else hq)[a:e], non_blocking=True)
                torch.cuda.current_stream().record_event()
        s1.wait_stream(s3)
        d2h(fine_d2h)
    return timed(f)


print(f"27 H2D copies over 2 streams + fine D2H: {h2d_two(True):.3f} ms; + 1 D2H copy: {h2d_two(False):.3f} ms")



def d2h_pieces(piece):
    with torch.cuda.stream(s2):
        for a, e in chunks(o_b):
            for x in range(a, e, piece):
                y = min(e, x + piece)
                ho[x:y].copy_(do[x:y], non_blocking=True)
            torch.cuda.current_stream().record_event()


def h2d_pieces(piece):
    with torch.cuda.stream(s1):
        half = kv_b // 2
        for a, e in ((0, half), (kv_b, kv_b + half), (half, kv_b), (kv_b + half, 2 * kv_b)):
            dk[a:e].copy_(hk[a:e], non_blocking=True)
            torch.cuda.current_stream().record_event()
        for a, e in chunks(q_b):
            for x in range(a, e, piece):
                y = min(e, x + piece)
                dq[x:y].copy_(hq[x:y], non_blocking=True)
            torch.cuda.current_stream().record_event()


for piece in (1 << 20, 2 << 20, 4 << 20):
    print(f"pipeline H2D + D2H chunks split in {piece >> 20} MB pieces: "
          f"{timed(lambda: (h2d(True), d2h_pieces(piece))):.3f} ms; both split: "
          f"{timed(lambda: (h2d_pieces(piece), d2h_pieces(piece))):.3f} ms")
