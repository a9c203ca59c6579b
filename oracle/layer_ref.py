"""oracle/layer_ref.py -- TEST INFRASTRUCTURE ONLY.

One Spava layer of REAL inputs through the reference's own operators (oracle/_ref: the
unmodified seqpar sources; or the C restatement, impl="c"), decomposed into independent
work items so it runs on every host core and so any subset of output rows can be
checked at full size:

* ("score", v, head)   score_context of one q-head against block v's kv-head
                       (score_block's loop body, simhost.cpp:209-224 -> approx.cpp:15-69);
                       the per-block total is the fp32 sum over heads in ascending order.
* select_essential per virtual block (approx.cpp:71-102) on those totals.
* ("anchor"|"block"|"query", ..., rows [r0, r1), head)  attention_lse of one head over a
  row slice (mha_lse's loop body, attention.cpp:158-178).  A row slice is an exact
  sub-problem: rows [r0, r1) of a block see [anchor | passing | own[0:r0) | own[r0:r1)
  causal], the same keys in the same order as the full block_attention call
  (approx.cpp:140-154), so each output row is bit-identical to the whole call's.
  Query partials (approx.cpp:156-188) are merged in host order (mha_merge,
  attention.cpp:180-197) per row.

Nothing in paper_2601_21444_b200/ imports this module; tests/ use it as the checker and
bench.py's reference arm / cpu_baseline time it (run_host's operator sequence minus
projections, simhost.cpp:328-426).
"""
from __future__ import annotations

import concurrent.futures as cf
import time

import numpy as np

from oracle import oracle as O


def geometry(n_v, n_t, hosts, l_a, l_p, zigzag=True):
    """split_context (partition.cpp:40-85) sizes; l_p clamped to l_b as resolve_lengths."""
    vh = 2 * hosts
    rem = n_v - l_a
    pad = (vh - rem % vh) % vh
    l_b = (rem + pad) // vh
    return dict(n_v=n_v, n_t=n_t, hosts=hosts, l_a=l_a, l_b=l_b, l_p=min(l_p, l_b), pad=pad,
                zigzag=zigzag)


def pair(g, h):
    """zigzag_map / naive_map virtual pair of physical host h (partition.cpp:9-29)."""
    H = g["hosts"]
    return (h, 2 * H - 1 - h) if g["zigzag"] else (2 * h, 2 * h + 1)


def valid_rows(g, v):
    """Non-pad rows of virtual block v (pads only at the tail of the last block)."""
    return g["l_b"] - (g["pad"] if v == 2 * g["hosts"] - 1 else 0)


def anchor_slice(g, h):
    """slice_anchor (partition.cpp:87-94)."""
    H, l_a = g["hosts"], g["l_a"]
    base, extra = l_a // H, l_a % H
    b = h * base + min(h, extra)
    return b, b + base + (1 if h < extra else 0)


class LayerRef:
    """Reference layer over global padded rows X = [anchor | 2H blocks | query] (fp32
    holding the bf16 values both paths consume).  Results are filled in lazily by run()."""

    def __init__(self, Q, K, V, g, hq, hkv, dh=128, impl="ref", designated=None):
        self.Q, self.K, self.V = Q, K, V
        self.g, self.hq, self.hkv, self.dh = g, hq, hkv, dh
        self.impl = impl if O.available(impl) else "c"
        self.scale = np.float32(1.0) / np.sqrt(np.float32(dh))
        H = g["hosts"]
        self.designated = H - 1 if designated is None else designated
        self.scores = {}      # v -> fp32 [l_b]
        self.parts = {}       # (v, head) -> fp32 [l_b]
        self.sel = {}         # v -> int32 global indices (ascending)
        self.out = {}         # (kind, key, head) -> {row: (out[dh], lse)}

    # -------------------------------------------------------------- geometry
    def block_rows(self, v):
        l_a, l_b = self.g["l_a"], self.g["l_b"]
        return l_a + v * l_b, l_a + (v + 1) * l_b

    def qrow(self):
        g = self.g
        return g["l_a"] + 2 * g["hosts"] * g["l_b"]

    def _cols(self, X, head, kv):
        c = (head // (self.hq // self.hkv) if kv else head) * self.dh
        return X[:, c:c + self.dh]

    def passing(self, v, head):
        """assemble_passing (approx.cpp:104-132): compressed rows of sources < v, source
        ascending, index ascending, of kv-head(head)."""
        if v == 0 or self.g["l_p"] == 0:
            return None, None
        rows = np.concatenate([self.sel[s] for s in range(v)])
        return (np.ascontiguousarray(self._cols(self.K[rows], head, True)),
                np.ascontiguousarray(self._cols(self.V[rows], head, True)))

    # ------------------------------------------------------------ work items
    def score_items(self, blocks=None):
        V2 = 2 * self.g["hosts"]
        blocks = range(V2) if blocks is None else blocks
        fl = 2 * self.g["n_t"] * self.g["l_b"] * self.dh
        return [("score", v, h, 0, 0, fl) for v in blocks for h in range(self.hq)]

    def attention_items(self, rows_anchor=(), rows_block=None, rows_query=(), m=16):
        """Row-slice x head items.  rows_block: {v: iterable of rows} (valid rows only)."""
        g, d = self.g, self.dh
        items = []

        def slices(rows):
            rows = sorted(set(int(r) for r in rows))
            i = 0
            while i < len(rows):
                j = i
                while j + 1 < len(rows) and rows[j + 1] == rows[j] + 1 and rows[j + 1] - rows[i] < m:
                    j += 1
                yield rows[i], rows[j] + 1
                i = j + 1

        for r0, r1 in slices(rows_anchor):
            fl = (4 * (r1 - r0) * r0 + 2 * (r1 - r0) ** 2) * d
            items += [("anchor", 0, h, r0, r1, fl) for h in range(self.hq)]
        for v, rows in (rows_block or {}).items():
            n_p = v * g["l_p"]
            for r0, r1 in slices(rows):
                fl = (4 * (r1 - r0) * (g["l_a"] + n_p + r0) + 2 * (r1 - r0) ** 2) * d
                items += [("block", v, h, r0, r1, fl) for h in range(self.hq)]
        for r0, r1 in slices(rows_query):
            for hh in range(g["hosts"]):
                a0, a1 = anchor_slice(g, hh)
                lo, hi = pair(g, hh)
                nk = (a1 - a0) + valid_rows(g, lo) + valid_rows(g, hi)
                self_ = hh == self.designated
                fl = (4 * (r1 - r0) * (nk + (r0 if self_ else 0)) + (2 * (r1 - r0) ** 2 if self_ else 0)) * d
                items += [("query", hh, h, r0, r1, fl) for h in range(self.hq)]
        return items

    def run_item(self, it):
        kind, key, head, r0, r1, _ = it
        g, d, impl, sc = self.g, self.dh, self.impl, float(self.scale)
        if kind == "score":
            b0, b1 = self.block_rows(key)
            nv = valid_rows(g, key)
            pad = None
            if nv < g["l_b"]:
                pad = np.zeros(g["l_b"], np.uint8)
                pad[nv:] = 1
            qr = self.qrow()
            q = np.ascontiguousarray(self._cols(self.Q[qr:qr + g["n_t"]], head, False))
            k = np.ascontiguousarray(self._cols(self.K[b0:b1], head, True))
            self.parts[(key, head)] = O.score_context(q, k, sc, pad, True, impl=impl)
            return it[5]
        segs = []
        if kind == "anchor":
            q = self._cols(self.Q[r0:r1], head, False)
            if r0:
                segs.append(dict(k=self._cols(self.K[:r0], head, True), v=self._cols(self.V[:r0], head, True)))
            segs.append(dict(k=self._cols(self.K[r0:r1], head, True), v=self._cols(self.V[r0:r1], head, True),
                             causal=True))
            allow = False
        elif kind == "block":
            b0, _ = self.block_rows(key)
            q = self._cols(self.Q[b0 + r0:b0 + r1], head, False)
            l_a = g["l_a"]
            if l_a:
                segs.append(dict(k=self._cols(self.K[:l_a], head, True), v=self._cols(self.V[:l_a], head, True)))
            kp, vp = self.passing(key, head)
            if kp is not None:
                segs.append(dict(k=kp, v=vp))
            if r0:
                segs.append(dict(k=self._cols(self.K[b0:b0 + r0], head, True),
                                 v=self._cols(self.V[b0:b0 + r0], head, True)))
            segs.append(dict(k=self._cols(self.K[b0 + r0:b0 + r1], head, True),
                             v=self._cols(self.V[b0 + r0:b0 + r1], head, True), causal=True))
            allow = True
        else:  # query partial of physical host `key` (approx.cpp:156-188)
            qr = self.qrow()
            q = self._cols(self.Q[qr + r0:qr + r1], head, False)
            a0, a1 = anchor_slice(g, key)
            if a1 > a0:
                segs.append(dict(k=self._cols(self.K[a0:a1], head, True), v=self._cols(self.V[a0:a1], head, True)))
            for v in pair(g, key):
                b0, _ = self.block_rows(v)
                nv = valid_rows(g, v)
                if nv > 0:
                    segs.append(dict(k=self._cols(self.K[b0:b0 + nv], head, True),
                                     v=self._cols(self.V[b0:b0 + nv], head, True)))
            if key == self.designated:
                if r0:
                    segs.append(dict(k=self._cols(self.K[qr:qr + r0], head, True),
                                     v=self._cols(self.V[qr:qr + r0], head, True)))
                segs.append(dict(k=self._cols(self.K[qr + r0:qr + r1], head, True),
                                 v=self._cols(self.V[qr + r0:qr + r1], head, True), causal=True))
            allow = True
        out, lse = O.attention_lse(np.ascontiguousarray(q), segs, sc, allow, impl=impl)
        self.out[(kind, key, head, r0)] = (out, lse)
        return it[5]

    def finish_scores(self, blocks=None):
        """score_block's ordered sum over heads, then select_essential (approx.cpp:71-102)."""
        g = self.g
        for v in (range(2 * g["hosts"]) if blocks is None else blocks):
            tot = np.zeros(g["l_b"], np.float32)
            for h in range(self.hq):
                tot = (tot + self.parts.pop((v, h))).astype(np.float32)
            self.scores[v] = tot
            self.sel[v] = O.select_essential(tot, g["l_p"], self.block_rows(v)[0], impl=self.impl)

    # ------------------------------------------------------------- results
    def rows(self, kind, key, rows):
        """Assembled [len(rows), hq*dh] outputs (and [len(rows), hq] lse) of computed rows."""
        rows = list(rows)
        out = np.zeros((len(rows), self.hq * self.dh), np.float32)
        lse = np.zeros((len(rows), self.hq), np.float32)
        starts = sorted(r0 for (k, kk, h, r0) in self.out if k == kind and kk == key and h == 0)
        for i, r in enumerate(rows):
            r0 = max(s for s in starts if s <= r)
            for h in range(self.hq):
                o, l = self.out[(kind, key, h, r0)]
                out[i, h * self.dh:(h + 1) * self.dh] = o[r - r0]
                lse[i, h] = l[r - r0]
        return out, lse

    def query_rows(self, rows):
        """Merged query rows (mha_merge over the hosts' partials, host order)."""
        parts = [self.rows("query", hh, rows) for hh in range(self.g["hosts"])]
        return O.mha_merge([p[0] for p in parts], [p[1] for p in parts], self.hq, self.dh, impl=self.impl)


def run_items(fn, items, threads, budget_s=None):
    """Run work items on `threads` host threads (ctypes releases the GIL), largest first;
    returns (seconds, flops done, items done).  budget_s stops issuing new items."""
    order = sorted(range(len(items)), key=lambda i: -items[i][5])
    t0 = time.perf_counter()
    done_fl, n_done = 0, 0
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        futs, nxt = set(), 0
        while nxt < len(order) and len(futs) < threads:
            futs.add(ex.submit(fn, items[order[nxt]]))
            nxt += 1
        while futs:
            fin, futs = cf.wait(futs, return_when=cf.FIRST_COMPLETED)
            for f in fin:
                done_fl += f.result()
                n_done += 1
                if nxt < len(order) and (budget_s is None or time.perf_counter() - t0 < budget_s):
                    futs.add(ex.submit(fn, items[order[nxt]]))
                    nxt += 1
    return time.perf_counter() - t0, done_fl, n_done


def layer_inputs(g, hq, hkv, dh=128, seed=1234):
    """The synthetic layer both arms consume: global padded rows [anchor | 2H blocks | query],
    N(0,1) rounded to bf16 (returned as fp32 carrying the bf16 values, pads zero).  Drawn
    with numpy's PCG64 from `seed` so the CPU reference and the GPU arm read the same bits."""
    H = g["hosts"]
    rows = g["l_a"] + 2 * H * g["l_b"] + g["n_t"]
    rng = np.random.default_rng(seed)

    def draw(w):
        x = rng.standard_normal((rows, w), dtype=np.float32)
        u = x.view(np.uint32)
        u += np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))  # bf16 nearest-even
        u &= np.uint32(0xFFFF0000)
        if g["pad"]:
            b = g["l_a"] + 2 * H * g["l_b"]
            x[b - g["pad"]:b] = 0.0
        return x

    return draw(hq * dh), draw(hkv * dh), draw(hkv * dh)


def host_rows(g, h):
    """Global row indices of physical host h's local buffer [anchor | lo | hi | query]."""
    l_a, l_b, H = g["l_a"], g["l_b"], g["hosts"]
    lo, hi = pair(g, h)
    q0 = l_a + 2 * H * l_b
    return np.concatenate([np.arange(l_a), np.arange(l_a + lo * l_b, l_a + (lo + 1) * l_b),
                           np.arange(l_a + hi * l_b, l_a + (hi + 1) * l_b), np.arange(q0, q0 + g["n_t"])])
