"""Core interactive protocols (reference: protocols/basic.py:1-239).

Same names, argument meaning, round counts, material consumption order and
ledger entries as the reference; every local step runs in a libmpx kernel.
In sim mode (``session.fused``) a round's mask, opening and finish collapse
into one kernel; in party mode the mask kernel's partial goes through an
NCCL collective before the finish kernel.
"""

from __future__ import annotations

import contextlib
import os

import numpy as np
import torch

from .. import _lib
from .. import kernels as K
from ..ring import bits_of_np, encode, encode_scalar
from ..sharing import AShare, BShare, add_public, public_bits_words
from ..session import arith_payload, bits_payload


def _check_same(x, y):
    if x.shape != y.shape:
        raise ValueError(f"shape mismatch {x.shape} vs {y.shape}")


def mul(session, x: AShare, y: AShare) -> AShare:
    """Element-wise Beaver product, one triple per element (basic.py:27-42)."""
    _check_same(x, y)
    if x.width != y.width:
        raise ValueError(f"width mismatch {x.width} vs {y.width}")
    w, n, L = x.width, x.size, session.L
    a, b, c = session.store.take_triples(w, n)
    z = session.alloc((L,) + x.shape)
    if session.fused:
        K.mul_fused(z, x.values, y.values, a.ptr, b.ptr, c.ptr, a.ps, L, n, w, session.p0)
        session.exchange(payload=2 * arith_payload(w, n))
    else:
        d, e = session.alloc((2, n)).unbind(0)          # one contiguous round payload
        K.mask_sub(d, x.values, a.ptr, a.ps, L, n, w)
        K.mask_sub(e, y.values, b.ptr, b.ps, L, n, w)
        d, e = session.exchange(arith=[(d, w), (e, w)])
        K.mul_finish(z, d, e, a.ptr, b.ptr, c.ptr, a.ps, L, n, w, session.p0)
    session.metrics.count(mul_count=1, mul_elems=n)
    return AShare(z, w, x.frac + y.frac, session.parties)


def matmul(session, x: AShare, y: AShare) -> AShare:
    return batch_matmul(session, [(x, y)])[0]


def batch_matmul(session, pairs) -> list[AShare]:
    """Independent matrix products in one round, one matrix triple each (basic.py:45-79).

    Z_l = C_l + D @ B_l + A_l @ E + [l==p0] D @ E, on the Z_2^64 GEMM kernels.
    Runs of equal-shape pairs whose operands sit at uniform strides (attention
    heads, Q/K/V on one input) are masked and reconstructed with one launch
    each; material order, the round and the ledger are per pair as in the
    reference.
    """
    L = session.L
    for x, y in pairs:
        if len(x.shape) != 2 or len(y.shape) != 2 or x.shape[1] != y.shape[0]:
            raise ValueError(f"bad matmul shapes {x.shape} @ {y.shape}")
    trip = []
    for x, y in pairs:
        m, k = x.shape
        trip.append(session.store.take_matrix_triple(x.width, m, k, y.shape[1]))
    groups = _groups(session, pairs, trip)
    masked = []
    fused_payload = 0
    unfused = [g for g in groups if not (_fused_tc(session, *_gshape(pairs, g)) or
                                          _fused_simt(session, *_gshape(pairs, g)))]
    # every masked D, E of the round in ONE buffer: party mode opens it with a
    # single collective, no concatenation. Canonical layout - all D's in pair
    # order, then all E's - so every party reduces the same element at the
    # same offset whatever its local launch grouping (_groups depends on its
    # own buffer addresses); a group's D's (E's) are still one run.
    nd = sum(len(g) * pairs[g[0]][0].size for g in unfused)
    arena = session.alloc((nd + sum(len(g) * pairs[g[0]][1].size for g in unfused),))
    at_d, at_e = 0, nd
    for g in groups:
        x0, y0 = pairs[g[0]]
        w, (m, k), r = x0.width, x0.shape, y0.shape[1]
        if g not in unfused:
            # sim mode: mask + open + limb split (or SIMT reconstruction) fused
            # below (one round, same logical payload as the reference's D, E openings)
            fused_payload += len(g) * (arith_payload(w, m * k) + arith_payload(w, k * r))
            continue
        D = arena[at_d:at_d + len(g) * m * k].view(len(g), m * k)
        at_d += len(g) * m * k
        E = arena[at_e:at_e + len(g) * k * r].view(len(g), k * r)
        at_e += len(g) * k * r
        _mask_group(D, [pairs[i][0].values for i in g], [trip[i][0] for i in g], L, m, k, w)
        _mask_group(E, [pairs[i][1].values for i in g], [trip[i][1] for i in g], L, k, r, w)
        for j in range(len(g)):
            masked += [(D[j], w), (E[j], w)]
    payload = sum(arith_payload(w, t.numel()) for t, w in masked) + fused_payload
    opened = session.exchange(arith=masked, payload=payload)
    out = [None] * len(pairs)
    pos = 0
    # sim mode: independent products of one round (e.g. a layer's dW and dX)
    # run on forked streams so small launches share the GPU; outputs are
    # allocated on the main stream, per-group scratch on its own stream
    conc = session.fused and len(groups) > 1 and CONCURRENT_GROUPS
    main = torch.cuda.current_stream(session.device) if conc else None
    used = []
    for gi, g in enumerate(groups):
        x0, y0 = pairs[g[0]]
        w, (m, k), r = x0.width, x0.shape, y0.shape[1]
        Zg = session.alloc((len(g), L, m, r))
        ctx = contextlib.nullcontext()
        if conc and gi > 0:
            st = _side_stream(session.device, gi - 1)
            st.wait_stream(main)
            used.append(st)
            ctx = torch.cuda.stream(st)
        with ctx:
            pos = _finish_group(session, pairs, trip, g, Zg, opened, pos, out, L)
    for st in used:
        main.wait_stream(st)
    return out


# off by default: measured no gain on the LeNet step (586.5 vs 589.8 steps/s)
# — the persistent GEMM holds every SM's shared memory, so nothing co-runs
CONCURRENT_GROUPS = os.environ.get("MPX_CONCURRENT_GROUPS", "0") != "0"
_SIDE: dict = {}


def _gshape(pairs, g):
    x0, y0 = pairs[g[0]]
    return x0.shape[0], x0.shape[1], y0.shape[1], x0.width


def _side_stream(device, i: int):
    key = (str(device), i)
    if key not in _SIDE:
        _SIDE[key] = torch.cuda.Stream(device)
    return _SIDE[key]


def _finish_group(session, pairs, trip, g, Zg, opened, pos, out, L) -> int:
    """Reconstruct one group's products into Zg; returns the next position in
    ``opened`` (the masked D, E of non-fused groups, in group order)."""
    x0, y0 = pairs[g[0]]
    w, (m, k), r = x0.width, x0.shape, y0.shape[1]
    if _fused_tc(session, m, k, r, w):
        if len(g) > 1:
            _beaver_matmul_fused_tc_group(session, Zg, [pairs[i] for i in g], [trip[i] for i in g], L, m, k, r,
                                          w)
        for j, i in enumerate(g):
            x, y = pairs[i]
            if len(g) == 1:
                A, B, C = trip[i]
                _beaver_matmul_fused_tc(session, Zg[j], x.values, y.values, A, B, C, L, m, k, r, w)
            session.metrics.count(matmul_count=1, matmul_macs=m * k * r)
            out[i] = AShare(Zg[j], w, x.frac + y.frac, session.parties)
        return pos
    if _fused_simt(session, m, k, r, w):
        _beaver_matmul_fused_simt(session, Zg, [pairs[i] for i in g], [trip[i] for i in g], L, m, k, r, w)
        for j, i in enumerate(g):
            x, y = pairs[i]
            session.metrics.count(matmul_count=1, matmul_macs=m * k * r)
            out[i] = AShare(Zg[j], w, x.frac + y.frac, session.parties)
        return pos
    Ds = opened[pos:pos + 2 * len(g):2]
    Es = opened[pos + 1:pos + 2 * len(g):2]
    pos += 2 * len(g)
    if not session.dry and _use_tc(m, k, r, w):
        for j, i in enumerate(g):
            A, B, C = trip[i]
            _beaver_matmul_tc(session, Zg[j], Ds[j], Es[j], A, B, C, L, m, k, r, w)
    else:
        A0, B0, C0 = trip[g[0]]
        Dg, Eg = _stacked(Ds, m * k), _stacked(Es, k * r)
        K.beaver_gemm_batched(Zg, m * r, L * m * r, C0.data_ptr(), C0.stride(0), _bstride(trip, g, 2),
                              Dg, Eg, A0.data_ptr(), A0.stride(0), _bstride(trip, g, 0),
                              B0.data_ptr(), B0.stride(0), _bstride(trip, g, 1), L, len(g), m, k, r,
                              session.p0, w)
    for j, i in enumerate(g):
        x, y = pairs[i]
        session.metrics.count(matmul_count=1, matmul_macs=m * k * r)
        out[i] = AShare(Zg[j], w, x.frac + y.frac, session.parties)
    return pos


def _ptr(t) -> int:
    return 0 if t.is_meta else t.data_ptr()


def _uniform(ptrs) -> int | None:
    """Common byte step of a pointer sequence (0 allowed), else None."""
    if len(ptrs) < 2:
        return 0
    d = ptrs[1] - ptrs[0]
    return d if all(ptrs[i + 1] - ptrs[i] == d for i in range(len(ptrs) - 1)) else None


def _layout(v):
    """('t' | 'r', party stride) of an operand the mask kernels read in place."""
    tps = K.transposed_base(v)
    if tps is not None:
        return "t", tps
    rps = K.rows_base(v)
    return ("r", rps) if rps is not None else (None, None)


def _groups(session, pairs, trip) -> list[list[int]]:
    """Consecutive equal-shape pairs whose x, y operands and triple parts sit
    at uniform strides (one launch per group); singletons otherwise."""
    groups: list[list[int]] = []
    for i, (x, y) in enumerate(pairs):
        if groups and not session.dry:
            g = groups[-1]
            x0, y0 = pairs[g[0]]
            same = (x.shape == x0.shape and y.shape == y0.shape and x.width == x0.width
                    and _layout(x.values) == _layout(x0.values) and _layout(y.values) == _layout(y0.values)
                    and _layout(x.values)[0] is not None and _layout(y.values)[0] is not None)
            if same:
                cand = g + [i]
                ok = all(_uniform([_ptr(pairs[j][s].values) for j in cand]) is not None for s in (0, 1)) and \
                    all(_uniform([_ptr(trip[j][s]) for j in cand]) is not None and
                        trip[cand[-1]][s].stride(0) == trip[g[0]][s].stride(0) for s in (0, 1, 2))
                if ok:
                    g.append(i)
                    continue
        groups.append([i])
    return groups


def _bstride(trip, g, s) -> int:
    return (_uniform([_ptr(trip[i][s]) for i in g]) or 0) // 8


def _stacked(ts, n):
    """[len(ts), n] view when the tensors are consecutive rows of one buffer."""
    if len(ts) == 1:
        return ts[0].reshape(1, n)
    base = ts[0]
    if all(_ptr(t) == _ptr(base) + 8 * n * j for j, t in enumerate(ts)) and not base.is_meta:
        return base.as_strided((len(ts), n), (n, 1))
    return torch.stack([t.reshape(n) for t in ts])


def _mask_group(out, vs, Ts, L, rows, cols, w):
    """out[j] = open(vs[j] - Ts[j]) (sim) / vs[j] - Ts[j] (party) for a group,
    one launch; transposed views (X^T, W^T, K^T) are read in place."""
    v0, T0 = vs[0], Ts[0]
    xbs = (_uniform([_ptr(v) for v in vs]) or 0) // 8
    abs_ = (_uniform([_ptr(T) for T in Ts]) or 0) // 8
    kind, ps = _layout(v0) if not v0.is_meta else ("r", rows * cols)
    if kind == "t":
        K.mask_sub_t(out, _ptr(v0), ps, _ptr(T0), T0.stride(0), L, rows, cols, w, batch=len(vs), x_bs=xbs,
                     a_bs=abs_)
    elif kind == "r":
        K.mask_sub_bs(out, _ptr(v0), ps, xbs, _ptr(T0), T0.stride(0), abs_, L, len(vs), rows * cols, w)
    else:
        for j, (v, T) in enumerate(zip(vs, Ts)):
            K.mask_sub(out[j], v.contiguous(), _ptr(T), T.stride(0), L, rows * cols, w)


def session_dry(v) -> bool:
    return v.is_meta


TC_MAX_WASTE = 2.2     # padded / useful MACs above which the SIMT kernel wins (conv1 fwd: 2.05 on TC)


# sim sessions (2..4 local parties) compare the tcgen05 path (mask+limb pass +
# GEMM) with the fused SIMT opening+reconstruction kernel, not with mask
# kernels + SIMT GEMM: LeNet conv1 forward (waste 2.05) is 116 vs 148 us on SIMT
SIM_TC_MAX_WASTE = 2.0


def _sim_waste(session) -> float:
    return SIM_TC_MAX_WASTE if 2 <= session.L <= 4 else TC_MAX_WASTE


def _use_tc(m, k, r, w=64, max_waste=None) -> bool:
    """tcgen05 limb GEMM when the padded work (128-row M tiles, 32/64-wide N
    tiles, 32/64/128-byte k-blocks) stays within TC_MAX_WASTE of the useful
    MACs; thin or tiny products go to the SIMT kernel."""
    if m < 96 or r < 16 or m * 2 * k * r < K.TC_MIN_MACS or (w != 64 and 2 * k > K.TC_MAX_K):
        return False
    waste = (K._rup(m, 128) / m) * (K.npad_tiles(r) / r) * (K.kpad(2 * k) / (2 * k))
    return waste <= (TC_MAX_WASTE if max_waste is None else max_waste)


def _fused_tc(session, m, k, r, w) -> bool:
    """Sim sessions run tcgen05-sized products as fused mask+limb split +
    split-operand GEMM, unless padding each K half separately (32 / 64 /
    128-byte k-blocks) costs much more MMA work than padding the concatenated
    2K (e.g. K = 10: 2 x 32 vs 32); up to 25% more MMA work is cheaper than
    the separate mask and limb passes (VGG K = 576: 2 x 640 vs 1152)."""
    return session.fused and 2 * K.kpad(k) <= 1.25 * K.kpad(2 * k) and _use_tc(m, k, r, w, _sim_waste(session))


def _fused_simt(session, m, k, r, w) -> bool:
    """Sim sessions with 2..4 local parties run the SIMT-sized products (thin
    outputs, long weight-gradient reductions) as one fused opening +
    reconstruction launch (D, E never materialised)."""
    return session.fused and 2 <= session.L <= 4 and not _use_tc(m, k, r, w, SIM_TC_MAX_WASTE)


def _beaver_matmul_fused_simt(session, Zg, pairs, trips, L, m, k, r, w):
    """Z_l = C_l + D @ (B_l + [l==p0] E) + A_l @ E for a group of equal-shape
    products (basic.py:66-75) with D = sum_l X_l - A_l, E = sum_l Y_l - B_l
    formed tile by tile inside the kernel; operand views read in place."""
    X0, Y0 = pairs[0][0].values, pairs[0][1].values
    A0, B0, C0 = trips[0]
    step = lambda ts: (_uniform([_ptr(t) for t in ts]) or 0) // 8  # noqa: E731
    x_js, y_js = step([p[0].values for p in pairs]), step([p[1].values for p in pairs])
    xps, xsr, xsc = _strides3(X0)
    yps, ysr, ysc = _strides3(Y0)
    if _thin_tc(len(pairs), L, m, k, r) and A0.stride(1) == k and B0.stride(1) == r and C0.stride(1) == r:
        K.beaver_tc_thin(Zg, m * r, C0.data_ptr(), C0.stride(0), _ptr(X0), xps, xsr, xsc, A0.data_ptr(),
                         A0.stride(0), _ptr(Y0), yps, ysr, ysc, B0.data_ptr(), B0.stride(0), L, m, k, r, session.p0, w)
        return
    if _long_tc(len(pairs), L, m, k, r, w) and A0.stride(1) == k and B0.stride(1) == r and C0.stride(1) == r:
        K.beaver_tc_long(Zg, m * r, C0.data_ptr(), C0.stride(0), _ptr(X0), xps, xsr, xsc, A0.data_ptr(),
                         A0.stride(0), _ptr(Y0), yps, ysr, ysc, B0.data_ptr(), B0.stride(0), L, m, k, r, session.p0, w)
        return
    K.beaver_gemm_sim(Zg, m * r, L * m * r, C0.data_ptr(), C0.stride(0), _bstride(trips, range(len(trips)), 2),
                      _ptr(X0), xps, xsr, xsc, x_js, A0.data_ptr(), A0.stride(0),
                      _bstride(trips, range(len(trips)), 0), _ptr(Y0), yps, ysr, ysc, y_js, B0.data_ptr(),
                      B0.stride(0), _bstride(trips, range(len(trips)), 1), L, len(pairs), m, k, r, session.p0, w)


# thin products (K, N <= 32: LeNet conv1 forward) on tcgen05 with the limb
# operands built in shared memory; MPX_THIN_TC=0 keeps them on the SIMT kernel
THIN_TC = os.environ.get("MPX_THIN_TC", "1") != "0"


def _thin_tc(batch, L, m, k, r) -> bool:
    return THIN_TC and batch == 1 and 2 <= L <= 3 and k <= 32 and r <= 32 and m >= 1024


# long-K small products (M, N <= 32: LeNet conv1 weight gradient) on tcgen05,
# split-K over the SMs; MPX_LONG_TC=0 keeps them on the SIMT kernel
LONG_TC = os.environ.get("MPX_LONG_TC", "1") != "0"
LONG_TC_MIN_K = 4096


def _long_tc(batch, L, m, k, r, w) -> bool:
    return LONG_TC and batch == 1 and k >= LONG_TC_MIN_K and K.long_tc_ok(L, m, k, r, w)


def _strides3(v):
    """(party, row, col) element strides of an [L, rows, cols] view."""
    if v.dim() != 3:
        raise ValueError("expected an [L, rows, cols] share view")
    return v.stride(0), v.stride(1), v.stride(2)


def _beaver_matmul_fused_tc(session, Z, X, Y, A, B, C, L, m, k, r, w):
    """All parties local: D = sum_l X_l - A_l and E = sum_l Y_l - B_l are
    never materialised as u64; one kernel per side writes their limb planes
    once (shared by every party's GEMM) next to the per-party material limbs
    (A_l; B_l + [l==p0] E), and the split-operand GEMM computes
    Z_l = C_l + [D | A_l] @ [B_l + [l==p0] E ; E] (basic.py:66-75)."""
    Mp, Np, Kh = K._rup(m, 128), K._rup(r, 32), K.kpad(k)
    dev = Z.device
    SA = torch.empty((8, Mp, Kh), dtype=torch.uint8, device=dev)
    PA = torch.empty((L, 8, Mp, Kh), dtype=torch.uint8, device=dev)
    SB = torch.empty((8, Np, Kh), dtype=torch.uint8, device=dev)
    PB = torch.empty((L, 8, Np, Kh), dtype=torch.uint8, device=dev)
    xps, xsr, xsc = _strides3(X)
    yps, ysk, ysn = _strides3(Y)
    # A side: logical (m, k); material A_l row-major m x k
    # B side: logical (r, k) = Y^T; material B_l row-major k x r (one launch for both sides)
    K.mask_limbs2(SA, PA, _ptr(X), xps, xsr, xsc, A.data_ptr(), A.stride(0), k, 1, m, Mp,
                  SB, PB, _ptr(Y), yps, ysn, ysk, B.data_ptr(), B.stride(0), 1, r, r, Np, L, k, Kh, session.p0, w)
    K.gemm_limbs_split(Z, PA, SA, PB, SB, L, m, r, Mp, Np, Kh, r, m * r, w, C.data_ptr(), C.stride(0))


def _beaver_matmul_fused_tc_group(session, Zg, pairs, trips, L, m, k, r, w):
    """A group of equal-shape products whose operands and triples sit at
    uniform strides (_groups): one mask+limb launch per side and one GEMM
    launch for all of them (batch = products x parties); per product exactly
    _beaver_matmul_fused_tc."""
    J = len(pairs)
    Mp, Np, Kh = K._rup(m, 128), K._rup(r, 32), K.kpad(k)
    dev = Zg.device
    SA = torch.empty((J, 8, Mp, Kh), dtype=torch.uint8, device=dev)
    PA = torch.empty((J, L, 8, Mp, Kh), dtype=torch.uint8, device=dev)
    SB = torch.empty((J, 8, Np, Kh), dtype=torch.uint8, device=dev)
    PB = torch.empty((J, L, 8, Np, Kh), dtype=torch.uint8, device=dev)
    X0, Y0 = pairs[0][0].values, pairs[0][1].values
    A0, B0, C0 = trips[0]
    step = lambda ts: (_uniform([_ptr(t) for t in ts]) or 0) // 8  # noqa: E731
    x_js, y_js = step([p[0].values for p in pairs]), step([p[1].values for p in pairs])
    a_js, b_js, c_js = step([t[0] for t in trips]), step([t[1] for t in trips]), step([t[2] for t in trips])
    xps, xsr, xsc = _strides3(X0)
    yps, ysk, ysn = _strides3(Y0)
    K.mask_limbs2(SA, PA, _ptr(X0), xps, xsr, xsc, A0.data_ptr(), A0.stride(0), k, 1, m, Mp,
                  SB, PB, _ptr(Y0), yps, ysn, ysk, B0.data_ptr(), B0.stride(0), 1, r, r, Np, L, k, Kh, session.p0, w,
                  jobs=J, x_js=x_js, a_js=a_js, y_js=y_js, b_js=b_js)
    K.gemm_limbs_split(Zg, PA, SA, PB, SB, J * L, m, r, Mp, Np, Kh, r, m * r, w, C0.data_ptr(), C0.stride(0),
                       zl=L, s_cin_j=c_js)


def _beaver_matmul_tc(session, Z, D, E, A, B, C, L, m, k, r, w):
    """Z_l += [D | A_l] @ [B_l + [l==p0] E ; E] as ONE tcgen05 limb GEMM per party
    (K doubled), so D@E at party 0 folds into its B operand (basic.py:72-75)."""
    Mp, Np, Kp = K._rup(m, 128), K._rup(r, 32), K.kpad(2 * k)
    A8 = torch.empty((L, 8, Mp, Kp), dtype=torch.uint8, device=Z.device)
    B8 = torch.empty((L, 8, Np, Kp), dtype=torch.uint8, device=Z.device)
    K.beaver_limbs(A8, B8, D, E, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), L, m, k, r, Mp, Np, Kp,
                   session.p0)
    K.gemm_limbs(Z, A8, B8, L, m, r, Mp, Np, Kp, r, m * r, False, w, cin=C.data_ptr(), s_cin=C.stride(0))


def and_gate(session, x: BShare, y: BShare) -> BShare:
    """Bitwise AND, one binary triple per bit (basic.py:82-95)."""
    _check_same(x, y)
    y = y.like_layout(x)
    L, rows, m = session.L, x.rows, x.m
    t = session.store.take_bin_triples(x.size)
    d, e = session.alloc((2, rows)).unbind(0)
    K.and_mask(d, e, x.words, y.words, t, L, rows, m)
    d, e = session.exchange(bits=[d, e], payload=2 * bits_payload(x.size))
    z = session.alloc(x.words.shape)
    K.and_finish(z, d, e, t, L, rows, m, session.p0)
    session.metrics.count(and_count=1, and_elems=x.size)
    return x._new(z)


def _carry_prefix(session, G: torch.Tensor, P: torch.Tensor, m: int, rows: int) -> None:
    """Kogge-Stone carries over the m-bit rows of G, P in place (basic.py:98-129).

    One AND round per level; level s consumes rows*2(m-s) bintriples laid
    out [G-part | P-part] per row (rows*(m-s) on the final level).
    """
    L = session.L
    s = 1
    while s < m:
        last = 2 * s >= m
        W = m - s
        cnt = rows * (W if last else 2 * W)
        t = session.store.take_bin_triples(cnt)
        if session.fused:
            K.carry_fused(G, P, t, L, rows, m, s, last, session.p0)
            session.exchange(payload=2 * bits_payload(cnt))
        else:
            pay = session.alloc((2 if last else 4, rows)).unbind(0)
            dg, eg = pay[0], pay[1]
            dp = None if last else pay[2]
            ep = None if last else pay[3]
            K.carry_mask(dg, eg, dp, ep, G, P, t, L, rows, m, s, last)
            parts = [dg, eg] if last else [dg, eg, dp, ep]
            got = session.exchange(bits=parts, payload=2 * bits_payload(cnt))
            if last:
                dg, eg = got
            else:
                dg, eg, dp, ep = got
            K.carry_finish(G, P, dg, eg, dp, ep, t, L, rows, m, s, last, session.p0)
        session.metrics.count(and_count=1, and_elems=cnt)
        s *= 2


def _sum_bits(session, P0, G, m, rows, like: BShare) -> BShare:
    out = session.alloc(P0.shape)
    K.sum_from_carries(out, P0, G, session.L, rows, m)
    return BShare(out, m, True, session.parties)


def public_add_bits(session, pub_bits, x: BShare) -> BShare:
    """Bits of (public + shared) mod 2^m; the generate layer is local (basic.py:139-152)."""
    if isinstance(pub_bits, torch.Tensor) and pub_bits.dtype == torch.int64:
        pub = pub_bits      # already row words
    else:
        pub = public_bits_words(pub_bits, x)
    x = x.as_rows()
    L, rows, m = session.L, x.rows, x.m
    G, P, P0 = (session.alloc(x.words.shape) for _ in range(3))
    K.pubadd_init(G, P, P0, pub, x.words, None, 0, 0, L, rows, m, session.p0)
    _carry_prefix(session, G, P, m, rows)
    return _sum_bits(session, P0, G, m, rows, x)


def binary_add(session, x: BShare, y: BShare) -> BShare:
    """Bits of (x + y) mod 2^m for two shared values (basic.py:155-161)."""
    g = and_gate(session, x.as_rows(), y.as_rows())
    p = x.as_rows() ^ y.as_rows()
    P0 = p.words
    P = P0.clone()
    G = g.words.clone()
    _carry_prefix(session, G, P, p.m, p.rows)
    return _sum_bits(session, P0, G, p.m, p.rows, p)


def _bit2a_round(session, b: BShare, width: int):
    L, rows, m = session.L, b.rows, b.m
    r_a, r_b = session.store.take_dabits(width, b.size)
    c = session.alloc((rows,))
    K.bit2a_mask(c, b.words, r_b.ptr, r_b.ps, r_b.bit, L, rows, m)
    (c,) = session.exchange(bits=[c], payload=bits_payload(b.size))
    session.metrics.count(bit2a_elems=b.size)
    return c, r_a


def bit2a(session, b: BShare, width: int) -> AShare:
    """XOR-shared bits -> additive shares in Z_2^width via daBits (basic.py:164-184)."""
    c, r_a = _bit2a_round(session, b, width)
    out = session.alloc((session.L,) + b.shape)
    K.bit2a_finish(out, c, r_a.ptr, r_a.ps, session.L, b.rows, b.m, width, session.p0, None, 0)
    return AShare(out, width, 0, session.parties)


def compose(session, bits: BShare, width: int, frac: int = 0) -> AShare:
    """sum_i 2^i * bit_i over the trailing axis, one round (basic.py:187-196).

    The per-bit conversions are reduced inside the finish kernel (no
    intermediate (..., m) tensor)."""
    bits = bits.as_rows()
    c, r_a = _bit2a_round(session, bits, width)
    out = session.alloc((session.L,) + bits.rows_shape)
    K.bit2a_finish(out, c, r_a.ptr, r_a.ps, session.L, bits.rows, bits.m, width, session.p0, None, 1)
    return AShare(out, width, frac, session.parties)


def decompose(session, x: AShare) -> BShare:
    """Bit decomposition (trailing axis of x.width bits) via a full-width edaBit
    (basic.py:199-214): open x - r, then add the public difference onto the
    shared bits of r with the carry tree."""
    w, n, L = x.width, x.size, session.L
    r_a, r_b = session.store.take_edabits(w, w, n)
    c = session.alloc((n,))
    K.mask_sub(c, x.values, r_a.ptr, r_a.ps, L, n, w)
    (c,) = session.exchange(arith=[(c, w)])
    G, P, P0 = (session.alloc((L,) + x.shape) for _ in range(3))
    K.pubadd_init(G, P, P0, c, None, r_b.ptr, r_b.ps, r_b.bit, L, n, w, session.p0)
    _carry_prefix(session, G, P, w, n)
    return _sum_bits(session, P0, G, w, n, None)


def gt(session, x: AShare, y: AShare) -> BShare:
    """Strict x > y: sign bit of y - x (basic.py:217-225)."""
    diff = y - x
    return decompose(session, diff)[..., diff.width - 1]


def const_share(session, value, width: int, frac: int, shape=()) -> AShare:
    """Fixed-point public constant as a degenerate sharing (basic.py:228-233)."""
    shape = tuple(shape)
    enc = encode(np.broadcast_to(np.asarray(value, np.float64), shape), width, frac, session.device)
    vals = session.alloc((session.L,) + shape)
    K.ring_lin(vals, None, 0, None, 0, 0, enc.reshape(-1) if enc.numel() else None,
               session.L, max(1, int(np.prod(shape))) if shape else 1, width, session.p0)
    return AShare(vals, width, frac, session.parties)


def add_const(session, x: AShare, value: float) -> AShare:
    """Add a public fixed-point constant at party 0 (basic.py:236-239)."""
    return add_public(x, encode_scalar(value, x.width, x.frac))
