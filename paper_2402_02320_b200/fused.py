"""Sim-mode whole-op fusion: record the material tape, launch one kernel.

When all parties live on this GPU (``SimSession``) the openings of a
non-linear function need no communication, so Exp / Log / Reciprocal run as
ONE kernel (csrc/fused_ops.cu). The exact sequence of dealer-material takes
is recorded by running the Python protocol once as a dry pass whose store
forwards every ``take_*`` to the real store (advancing the real cursors, as
the per-round path would) and logs the resulting views; the same pass
records the op/communication ledger into the live session's metrics. The
kernel then consumes the tape in order. Bit-exactness against the per-round
path and the reference is covered by tests/test_gpu_parity.py and
tests/test_fused_ops.py.
"""

from __future__ import annotations

import ctypes
import os
import math

import torch

from . import _lib
from .preprocessing import ArithMat, BitMat, BitTriples
from .ring import encode_scalar
from .sharing import AShare

TAPE_MAX = 160


class MatRef(ctypes.Structure):
    _fields_ = [("p0", ctypes.c_void_p), ("p1", ctypes.c_void_p), ("p2", ctypes.c_void_p),
                ("ps0", ctypes.c_int64), ("ps1", ctypes.c_int64), ("ps2", ctypes.c_int64),
                ("off", ctypes.c_int64), ("kind", ctypes.c_int), ("per0", ctypes.c_int),
                ("per1", ctypes.c_int), ("pad", ctypes.c_int)]


class Tape(ctypes.Structure):
    _fields_ = [("m", MatRef * TAPE_MAX), ("n", ctypes.c_int)]


class TourLevels(ctypes.Structure):
    _fields_ = [("start", ctypes.c_int * 17), ("nlev", ctypes.c_int)]


class SoftmaxSegs(ctypes.Structure):
    _fields_ = [("resc", ctypes.c_int), ("lev", ctypes.c_int * 17), ("nlev", ctypes.c_int),
                ("attexp", ctypes.c_int), ("recip", ctypes.c_int), ("end", ctypes.c_int),
                ("log2e_p", ctypes.c_uint64), ("p", ctypes.c_int), ("w32", ctypes.c_int)]


class FusedParams(ctypes.Structure):
    _fields_ = [("w", ctypes.c_int), ("p", ctypes.c_int), ("iters", ctypes.c_int), ("bias", ctypes.c_int),
                ("c", ctypes.c_int), ("L", ctypes.c_int), ("p0", ctypes.c_int),
                ("log2e_p", ctypes.c_uint64), ("bias_2p", ctypes.c_uint64), ("one_p", ctypes.c_uint64),
                ("m1_p", ctypes.c_uint64), ("ln2_p", ctypes.c_uint64), ("coef_p", ctypes.c_uint64 * 5),
                ("coef0_2p", ctypes.c_uint64), ("coef_nz", ctypes.c_int * 5), ("pf", ctypes.c_int)]


def _take_ref(store, method: str, args: tuple, n: int) -> tuple:
    """Perform one take on the real store; return its MatRef fields (``n`` =
    elements of the fused op, so per-element strides are count // n)."""
    if method == "take_triples":
        a, b, c = store.take_triples(*args)
        return (a.ptr, b.ptr, c.ptr, a.ps, b.ps, c.ps, 0, 0, args[1] // n, 0, 0)
    if method == "take_bin_triples":
        t = store.take_bin_triples(*args)
        return (t.a_ptr, t.b_ptr, t.c_ptr, t.ps, t.ps, t.ps, t.bit, 1, args[0] // n, 0, 0)
    if method == "take_dabits":
        ra, rb = store.take_dabits(*args)
        per = args[1] // n
        return (ra.ptr, rb.ptr, 0, ra.ps, rb.ps, 0, rb.bit, 2, per, per, 0)
    if method == "take_edabits":
        ra, rb = store.take_edabits(*args)
        per = args[2] // n
        return (ra.ptr, rb.ptr if rb else 0, 0, ra.ps, rb.ps if rb else 0, 0, rb.bit if rb else 0, 2, per,
                per * args[1] if rb else 0, 0)
    raise NotImplementedError(f"{method} is not fused")


class TapeStore:
    """Dry-run store that forwards takes to the real store and logs them."""

    dry = True

    def __init__(self, real, n: int):
        self.real = real
        self.n = n
        self.parties = real.parties
        self.n_parties = real.n_parties
        self.tape: list[tuple] = []
        self.calls: list[tuple] = []

    @property
    def L(self):
        return len(self.parties)

    def _m(self, *shape):
        return torch.empty(shape, dtype=torch.int64, device="meta")

    def _rec(self, method, args):
        self.calls.append((method, args))
        self.tape.append(_take_ref(self.real, method, args, self.n))

    def take_triples(self, width, count):
        self._rec("take_triples", (width, count))
        return tuple(ArithMat(self._m(self.L, count)) for _ in range(3))

    def take_bin_triples(self, count):
        self._rec("take_bin_triples", (count,))
        z = self._m(self.L, 1)
        return BitTriples(z, z, z, 0)

    def take_dabits(self, width, count):
        self._rec("take_dabits", (width, count))
        return ArithMat(self._m(self.L, count)), BitMat(self._m(self.L, 1), 0)

    def take_edabits(self, width, m, count, need_bits: bool = True):
        self._rec("take_edabits", (width, m, count, need_bits))
        return ArithMat(self._m(self.L, count)), (BitMat(self._m(self.L, 1), 0) if need_bits else None)

    def take_matrix_triple(self, width, m, k, r):
        raise NotImplementedError("matrix triples are not fused")


def _merge_metrics(dst, src) -> None:
    """Add a scoped ledger recorded from an empty scope stack under dst's
    current scope path."""
    from .metrics import OpCounters
    prefix = "/".join(dst._stack)
    for key, e in src.ledger.items():
        full = (prefix or "(root)") if key == "(root)" else (f"{prefix}/{key}" if prefix else key)
        entry = dst.ledger.get(full)
        if entry is None:
            entry = dst.ledger[full] = OpCounters()
        entry.add(e)
    dst.total.add(src.total)
    for peer, b in src.bytes_per_peer.items():
        dst.bytes_per_peer[peer] += b
    dst.physical_bytes += src.physical_bytes


# (kind, shape, width, frac, params, L, n, p0) -> (take calls, ledger, out width, out frac)
_SCHEDULES: dict = {}


_ENTRY = {"reciprocal": "mpx_reciprocal_fused", "exp": "mpx_exp_fused", "log": "mpx_log_fused",
          "attexp": "mpx_attexp_fused"}
_SIG_SET = False


def _bind():
    global _SIG_SET
    lib = _lib.load()
    if not _SIG_SET:
        for nm in _ENTRY.values():
            fn = getattr(lib, nm)
            fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_void_p]
            fn.restype = ctypes.c_int
        for nm in ("mpx_relu_fused", "mpx_maxlevel_fused"):
            fn = getattr(lib, nm)
            fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_void_p]
            fn.restype = ctypes.c_int
        lib.mpx_maxtour_fused.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.mpx_maxtour_fused.restype = ctypes.c_int
        lib.mpx_fused_tour_size.argtypes = [ctypes.POINTER(ctypes.c_int64)]
        tsz = ctypes.c_int64()
        lib.mpx_fused_tour_size(ctypes.byref(tsz))
        if tsz.value != ctypes.sizeof(TourLevels):
            raise _lib.MpxError(f"fused tournament ABI mismatch: C {tsz.value} vs ctypes {ctypes.sizeof(TourLevels)}")
        lib.mpx_softmax_fused.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64, ctypes.c_int] + \
            [ctypes.c_void_p] * 6
        lib.mpx_softmax_fused.restype = ctypes.c_int
        lib.mpx_fused_softmax_size.argtypes = [ctypes.POINTER(ctypes.c_int64)]
        ssz = ctypes.c_int64()
        lib.mpx_fused_softmax_size(ctypes.byref(ssz))
        if ssz.value != ctypes.sizeof(SoftmaxSegs):
            raise _lib.MpxError(f"fused softmax ABI mismatch: C {ssz.value} vs ctypes {ctypes.sizeof(SoftmaxSegs)}")
        lib.mpx_fused_abi_sizes.argtypes = [ctypes.POINTER(ctypes.c_int64)] * 4
        sizes = [ctypes.c_int64() for _ in range(4)]
        lib.mpx_fused_abi_sizes(*[ctypes.byref(s) for s in sizes])
        want = (ctypes.sizeof(MatRef), ctypes.sizeof(Tape), ctypes.sizeof(FusedParams), TAPE_MAX)
        if tuple(s.value for s in sizes) != want:
            raise _lib.MpxError(f"fused ABI layout mismatch: C {[s.value for s in sizes]} vs ctypes {want}")
        _SIG_SET = True
    return lib


def material_bytes(calls, L: int) -> int:
    """Dealer bytes a fused op must read for one call (all L local parties)."""
    tot = 0
    for method, args in calls:
        if method == "take_triples":
            tot += 3 * 8 * args[1]
        elif method == "take_bin_triples":
            tot += 3 * args[0] / 8
        elif method == "take_dabits":
            tot += 8 * args[1] + args[1] / 8
        elif method == "take_edabits":
            tot += 8 * args[2] + (args[2] * args[1] / 8 if args[3] else 0)
    return int(tot * L)


def fusable(session, x: AShare) -> bool:
    return (getattr(session, "fused", False) and getattr(session, "fuse_ops", True)
            and x.width == 64 and (1 <= session.L <= 4 or session.L == 8) and 2 * x.frac <= 62 and x.size > 0)


def fusable_attexp(session, x: AShare) -> bool:
    """attention_exp kernel: w32 input -> w64 output; the converted segment
    (p + clog2(p) + 1 bits) fits the narrow word and 2p <= 62."""
    p = x.frac
    return (getattr(session, "fused", False) and getattr(session, "fuse_ops", True)
            and x.width == 32 and (1 <= session.L <= 4 or session.L == 8) and x.size > 0 and 1 <= p <= 31
            and p + max(1, (p - 1).bit_length()) + 1 <= 32)


def fusable_cmp(session, x: AShare) -> bool:
    """ReLU / max-level kernels: any ring width >= 8."""
    return (getattr(session, "fused", False) and getattr(session, "fuse_ops", True)
            and 8 <= x.width <= 64 and (1 <= session.L <= 4 or session.L == 8) and x.size > 0)


# Reciprocal / Exp / Log / attention-exp calls of at most this many elements
# (softmax row sums, LeNet's 128 x 10 logits, attention scores) prefetch each
# element's whole take list to L2 before the first round: they are chains of
# dependent rounds on a few CTAs, not bandwidth-bound (env MPX_PF_SMALL).
PF_SMALL_ELEMS = int(os.environ.get("MPX_PF_SMALL", "0"))  # measured neutral: off


def params_for(kind: str, session, x: AShare, params) -> FusedParams:
    w, p = x.width, x.frac
    P = FusedParams()
    P.w, P.p, P.L, P.p0 = w, p, session.L, session.p0
    P.pf = int(x.size <= PF_SMALL_ELEMS)
    P.iters = params.newton_iters
    coeffs = None
    if kind == "exp":
        P.bias = min(p, 38 - p)
        P.c = max(1, (w - p - 1 - 1).bit_length())
        P.log2e_p = encode_scalar(math.log2(math.e), w, p)
        P.bias_2p = encode_scalar(float(P.bias), w, 2 * p)
        coeffs = params.exp_coeffs
    elif kind == "attexp":
        sq = params.exp_square
        delta = math.log2(params.exp_coeffs[4]) + sq.lead_shift
        P.c = max(1, (p - 1).bit_length())
        P.bias = sq.lead_shift
        P.coef_p[0] = encode_scalar(float(p) + delta, w, p)
        P.coef_p[1] = encode_scalar(sq.t3, 64, p)
        P.coef_p[2] = encode_scalar(sq.t2, 64, p)
        P.coef_p[3] = encode_scalar(sq.lead * sq.t1, 64, p)
        P.coef0_2p = encode_scalar(sq.lead * sq.t0, 64, 2 * p)
        return P
    elif kind == "log":
        P.m1_p = encode_scalar(-1.0, w, p)
        P.ln2_p = encode_scalar(math.log(2.0), w, p)
        coeffs = params.log_coeffs
    P.one_p = encode_scalar(1.0, w, p)
    if coeffs is not None:
        if len(coeffs) != 5:
            raise ValueError("fused kernels evaluate degree-4 polynomials")
        for i in range(1, 5):
            P.coef_p[i] = encode_scalar(coeffs[i], w, p)
            P.coef_nz[i] = int(coeffs[i] != 0)
        P.coef0_2p = encode_scalar(float(coeffs[0]), w, 2 * p)
    return P


def _schedule(kind: str, session, key, n_elems: int, protocol, metas):
    """Take schedule + ledger for one fused call: recorded by a dry pass of the
    Python protocol over the real store the first time, replayed afterwards."""
    from .metrics import CommMetrics
    from .session import SimSession
    sched = _SCHEDULES.get(key)
    if sched is None:
        store = TapeStore(session.store, n_elems)
        tmp = CommMetrics(session.metrics.party, session.n_parties)
        ts = SimSession(session.n_parties, store, metrics=tmp)
        ym = protocol(ts, *metas)
        if len(store.tape) > TAPE_MAX:
            raise _lib.MpxError(f"{kind}: tape of {len(store.tape)} takes exceeds {TAPE_MAX}")
        ym = ym[0] if isinstance(ym, tuple) else ym
        sched = (tuple(store.calls), tmp, ym.width, ym.frac)
        _SCHEDULES[key] = sched
        entries = store.tape
    else:
        entries = [_take_ref(session.store, m, a, n_elems) for m, a in sched[0]]
    _merge_metrics(session.metrics, sched[1])
    tape = Tape()
    for i, ent in enumerate(entries):
        tape.m[i] = MatRef(*ent)
    tape.n = len(entries)
    return tape, sched


def _meta(x: AShare) -> AShare:
    return AShare(torch.empty(x.values.shape, dtype=torch.int64, device="meta"), x.width, x.frac, x.parties)


def _launch(lib, entry, args, prof_info):
    _lib.LAUNCHES += 1
    prof = _lib.profiling()
    if prof is not None:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
    rc = getattr(lib, entry)(*args, _lib.stream_ptr())
    if prof is not None:
        ev1.record()
        prof.append((entry, prof_info, ev0, ev1))
    if rc != 0:
        raise _lib.MpxError(f"{entry} returned {rc}")


def run_fused(kind: str, session, x: AShare, params, protocol) -> AShare:
    """Launch the fused kernel for ``protocol`` on ``x`` (Reciprocal/Exp/Log)."""
    lib = _bind()
    key = (kind, x.shape, x.width, x.frac, params, session.L, session.n_parties, session.p0)
    tape, (calls, _, out_w, out_f) = _schedule(kind, session, key, x.size, protocol, (_meta(x),))
    P = params_for(kind, session, x, params)
    y = session.alloc(x.values.shape)
    xv = x.values.contiguous()
    _launch(lib, _ENTRY[kind], (y.data_ptr(), xv.data_ptr(), x.size, ctypes.addressof(tape), ctypes.addressof(P)),
            (kind, x.size, session.L, calls, 2))
    return AShare(y, out_w, out_f, session.parties)


# 1: the ReLU / max-level kernels pull each element's whole take list towards
# L2 before the first round (latency-bound carry chains); env MPX_PF_CMP=0 off.
PREFETCH_CMP = int(os.environ.get("MPX_PF_CMP", "1"))


def _basic_params(session, x: AShare) -> FusedParams:
    P = FusedParams()
    P.w, P.p, P.L, P.p0 = x.width, x.frac, session.L, session.p0
    P.pf = PREFETCH_CMP
    return P


def relu_fused(session, x: AShare, protocol, want_sign: bool):
    """ReLU in one kernel: (y, converted sign or None)."""
    lib = _bind()
    key = ("relu", x.shape, x.width, x.frac, session.L, session.n_parties, session.p0)
    tape, (calls, _, out_w, out_f) = _schedule("relu", session, key, x.size, protocol, (_meta(x),))
    P = _basic_params(session, x)
    y = session.alloc(x.values.shape)
    sg = session.alloc(x.values.shape) if want_sign else None
    _launch(lib, "mpx_relu_fused", (y.data_ptr(), sg.data_ptr() if sg is not None else None,
                                    x.values.contiguous().data_ptr(), x.size, ctypes.addressof(tape),
                                    ctypes.addressof(P)), ("relu", x.size, session.L, calls, 3 if want_sign else 2))
    out = AShare(y, out_w, out_f, session.parties)
    return out, (AShare(sg, x.width, 0, session.parties) if sg is not None else None)


def maxlevel_fused(session, u: AShare, v: AShare, protocol) -> AShare:
    """One max_vec tournament level in one kernel: v + bit2a(gt(u, v)) * (u - v)."""
    lib = _bind()
    key = ("maxlevel", u.shape, u.width, u.frac, session.L, session.n_parties, session.p0)
    tape, (calls, _, out_w, out_f) = _schedule("maxlevel", session, key, u.size, protocol, (_meta(u), _meta(v)))
    P = _basic_params(session, u)
    y = session.alloc(u.values.shape)
    _launch(lib, "mpx_maxlevel_fused", (y.data_ptr(), u.values.contiguous().data_ptr(),
                                        v.values.contiguous().data_ptr(), u.size, ctypes.addressof(tape),
                                        ctypes.addressof(P)), ("maxlevel", u.size, session.L, calls, 3))
    return AShare(y, out_w, out_f, session.parties)


def tour_fusable(session, x: AShare) -> bool:
    d = x.shape[-1] if x.shape else 0
    return fusable_cmp(session, x) and 2 <= d <= 512


def maxtour_fused(session, x: AShare, protocol) -> AShare:
    """A whole max_vec tournament in one kernel (one CTA per row). Each level's
    takes are scheduled exactly as the per-level path would (same keys, same
    order), then concatenated into one tape."""
    lib = _bind()
    d0 = x.shape[-1]
    rows = x.size // d0
    lead = x.shape[:-1]
    entries, lev_start = [], []
    d = d0
    mu = None
    while d > 1:
        half = d // 2
        shp = lead + (half,)
        mu = AShare(torch.empty((session.L,) + shp, dtype=torch.int64, device="meta"), x.width, x.frac,
                    x.parties)
        key = ("maxlevel", shp, x.width, x.frac, session.L, session.n_parties, session.p0)
        tape, _ = _schedule("maxlevel", session, key, rows * half, protocol, (mu, mu))
        lev_start.append(len(entries))
        entries += [tape.m[i] for i in range(tape.n)]
        d = half + (d - 2 * half)
    if len(entries) > TAPE_MAX or len(lev_start) > 16:
        raise _lib.MpxError(f"max tournament of width {d0}: {len(entries)} takes exceed the tape")
    tape = Tape()
    for i, m in enumerate(entries):
        tape.m[i] = m
    tape.n = len(entries)
    lv = TourLevels()
    for i, s in enumerate(lev_start):
        lv.start[i] = s
    lv.start[len(lev_start)] = len(entries)
    lv.nlev = len(lev_start)
    P = _basic_params(session, x)
    y = session.alloc((session.L,) + lead)
    _launch(lib, "mpx_maxtour_fused", (y.data_ptr(), x.values.contiguous().data_ptr(), rows, d0,
                                       ctypes.addressof(tape), ctypes.addressof(lv), ctypes.addressof(P)),
            ("maxtour", rows, session.L, None, 0))
    return AShare(y, x.width, x.frac, session.parties)


SOFTMAX_FUSED_MAX_ROWS = int(os.environ.get("MPX_SOFTMAX_FUSED_ROWS", "296"))   # 2 CTAs x 148 SMs


def softmax_fusable(session, x: AShare, cast_width) -> bool:
    """One-kernel softmax_parts: 64-bit input narrowed to 32 bits, rows of
    2..256 (one CTA per row), and the attention-exp / reciprocal kernels'
    own conditions on the narrowed values / row sums."""
    if not x.shape or cast_width != 32 or x.width != 64:
        return False
    d = x.shape[-1]
    if not (2 <= d <= 256 and fusable_cmp(session, x)):
        return False
    # one CTA per row runs every stage's chain of rounds back to back (the
    # reciprocal on one thread): a win only when all rows are resident at once
    # (LeNet's 128 logit rows); the attention's 1024 rows would take several
    # waves of the whole chain (measured 3.82 vs 3.33 ms per Transformer
    # forward), so they keep the per-stage kernels.
    if x.size // d > SOFTMAX_FUSED_MAX_ROWS:
        return False
    narrow_meta = AShare(torch.empty((session.L,) + x.shape, dtype=torch.int64, device="meta"), 32, x.frac,
                         x.parties)
    return fusable_attexp(session, narrow_meta) and fusable(session, x)


def softmax_fused(session, x: AShare, params, base2: bool, protocols):
    """softmax_parts (nn.py:115-136) in ONE kernel, one CTA per row. Each
    stage's takes are scheduled exactly as the standalone fused kernels
    schedule them (same keys, same scopes, same order) and concatenated into
    one tape, so material use and the ledger equal the per-op path.
    ``protocols``: (rescale, max_level, attention_exp, reciprocal) callables
    for the dry passes. Returns (e, r)."""
    lib = _bind()
    rescale, max_level, att, recip = protocols
    p, L = x.frac, session.L
    d0 = x.shape[-1]
    lead = x.shape[:-1]
    rows = x.size // d0
    meta = lambda shape, w, f: AShare(torch.empty((L,) + tuple(shape), dtype=torch.int64, device="meta"), w, f,  # noqa: E731
                                      x.parties)
    entries = []
    sg = SoftmaxSegs()
    sg.resc = -1
    if not base2:
        with session.scope("rescale"):
            key = ("softmax_rescale", x.shape, x.width, p, L, session.n_parties, session.p0)
            tape, _ = _schedule("softmax_rescale", session, key, x.size, rescale, (meta(x.shape, 64, p),))
            sg.resc = len(entries)
            entries += [tape.m[i] for i in range(tape.n)]
    with session.scope("maxcut"):
        d, nlev = d0, 0
        while d > 1:
            half = d // 2
            shp = lead + (half,)
            mu = meta(shp, 32, p)
            key = ("maxlevel", shp, 32, p, L, session.n_parties, session.p0)
            tape, _ = _schedule("maxlevel", session, key, rows * half, max_level, (mu, mu))
            sg.lev[nlev] = len(entries)
            nlev += 1
            entries += [tape.m[i] for i in range(tape.n)]
            d = half + (d - 2 * half)
        sg.nlev = nlev
    with session.scope("exp"):
        xm = meta(x.shape, 32, p)
        key = ("attexp", x.shape, 32, p, params, L, session.n_parties, session.p0)
        tape, (_, _, ew, ef) = _schedule("attexp", session, key, x.size, att, (xm,))
        sg.attexp = len(entries)
        entries += [tape.m[i] for i in range(tape.n)]
        Pe = params_for("attexp", session, xm, params)
    with session.scope("sum_recip"):
        rm = meta(lead, ew, ef)
        key = ("reciprocal", tuple(lead), ew, ef, params, L, session.n_parties, session.p0)
        tape, (_, _, rw, rf) = _schedule("reciprocal", session, key, rows, recip, (rm,))
        sg.recip = len(entries)
        entries += [tape.m[i] for i in range(tape.n)]
        Pr = params_for("reciprocal", session, rm, params)
    sg.end = len(entries)
    if len(entries) > TAPE_MAX:
        raise _lib.MpxError(f"softmax of width {d0}: {len(entries)} takes exceed the tape")
    tp = Tape()
    for i, m in enumerate(entries):
        tp.m[i] = m
    tp.n = len(entries)
    sg.log2e_p = encode_scalar(math.log2(math.e), 64, p)
    sg.p, sg.w32 = p, 32
    Pm = _basic_params(session, meta(x.shape, 32, p))
    Pe.pf = Pr.pf = 0
    e = session.alloc((L,) + x.shape)
    r = session.alloc((L,) + tuple(lead))
    _launch(lib, "mpx_softmax_fused", (e.data_ptr(), r.data_ptr(), x.values.contiguous().data_ptr(), rows, d0,
                                       ctypes.addressof(tp), ctypes.addressof(sg), ctypes.addressof(Pm),
                                       ctypes.addressof(Pe), ctypes.addressof(Pr)), ("softmax", rows, L, None, 0))
    return AShare(e, ew, ef, session.parties), AShare(r, rw, rf, session.parties)
