#!/usr/bin/env python
"""Benchmark: secure LeNet training steps/s (BASELINE.json configs[1]) on B200,
plus the cfg-5 party-scaling sweep (Reciprocal / Exp / Log on 2^24 elements,
Beaver matmul 4096^2) and the Simple-MLP training step (configs[0]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

* N = 1: the 1-GPU all-parties-simulated run: 3 parties on cuda:0, each
  training step captured once in a CUDA graph and replayed.
* N > 1 (torchrun, one rank per GPU): N parties, one per GPU, openings over
  NCCL, eager steps.
* ``--impl reference``: the UNMODIFIED reference package, pip-installed in
  ``baseline/_ref`` (git-ignored, travels to the GPU box with the repo), run
  through its own API by ``baseline/reference_arm.py`` on all host cores:
  same metric and config, the batch split over the cores (the oracle port
  under ``oracle/`` only if the install is missing).

A step = one secure SGD step of LeNet (forward, softmax-CE, backward, update)
on a batch of 128 synthetic 28x28 images, weights secret-shared. The trusted
dealer (on-device Philox, bit-exact with the reference's numpy dealer)
re-deals fresh single-use material before every step outside the timed
region (reported as dealer_ms_per_step; the paper times the online phase).
Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import multiprocessing as mp
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "secure CNN train steps/s: LeNet, batch 128 (BASELINE configs[1])"
LENET_WORKLOAD = ("configs[1]: secure LeNet training step (conv20-5x5, avgpool, ReLU, conv50-5x5, avgpool, ReLU, "
                  "FC800x500, ReLU, FC500x10; softmax-CE; SGD lr 2^-5)")
UNIT = "steps/s"
RECIP_UNIT = "elements/s"
BATCH = 128
LR_SHIFT = 5
SEED = 7
FRAC = 23
WIDTH = 64


def label_key(label: str):
    """scenarios.py:48-51: Philox key = sha256(f"{seed}:{label}")[:16] as two LE u64."""
    tag = hashlib.sha256(f"{SEED}:{label}".encode()).digest()
    return [int.from_bytes(tag[:8], "little"), int.from_bytes(tag[8:16], "little")]


def workload_inputs(n_elems: int) -> np.ndarray:
    """x = +-2^U(-8, 8), random sign (SURVEY §8d cfg 5), deterministic."""
    rng = np.random.default_rng(20240202)
    mags = np.exp2(rng.uniform(-8.0, 8.0, n_elems))
    return mags * rng.choice(np.array([-1.0, 1.0]), n_elems)


def encode_np(x, width=WIDTH, frac=FRAC):
    s = np.floor(np.asarray(x, dtype=np.float64) * float(1 << frac)).astype(np.int64)
    return s.view(np.uint64)


# ---------------------------------------------------------------------------
# CPU reference arm / cpu_baseline: the oracle port, one process per core


def _cpu_worker(args):
    chunk, n_parties, seed = args
    import oracle as O
    xs = workload_inputs(chunk)
    enc = encode_np(xs)

    def fn(s):
        x = O.AShare(O.deal_inputs_arith(enc, n_parties, WIDTH, label_key("share:x")), WIDTH, FRAC)
        return O.reciprocal(s, x)

    dry = O.Sim(n_parties, O.Demand(n_parties))
    fn(dry)
    live = O.Sim(n_parties, O.Store(seed, n_parties, dry.store.demands))
    x = O.AShare(O.deal_inputs_arith(enc, n_parties, WIDTH, label_key("share:x")), WIDTH, FRAC)
    t0 = time.perf_counter()
    O.reciprocal(live, x)
    return time.perf_counter() - t0


def cpu_reference(sample: int, n_parties: int, cores: int | None = None, reps: int = 1):
    """Online reciprocal on `sample` elements split over all host cores.
    Returns (elements/s, cores, seconds)."""
    cores = cores or os.cpu_count() or 1
    chunk = max(1024, sample // cores)
    tasks = [(chunk, n_parties, 11 + i) for i in range(cores)]
    ctx = mp.get_context("fork")
    best = None
    with ctx.Pool(cores) as pool:
        for _ in range(reps):
            t0 = time.perf_counter()
            times = pool.map(_cpu_worker, tasks)
            wall = time.perf_counter() - t0
            online = max(times)  # all workers run concurrently; slowest bounds
            rate = chunk * cores / online
            best = rate if best is None else max(best, rate)
    return best, cores, online


def lenet_data(B: int, seed: int = 11):
    """SURVEY §8d cfg 2: x ~ U(0,1) 28x28x1, labels uniform in 0..9 (one-hot)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(0.0, 1.0, (B, 1, 28, 28)), np.eye(10)[rng.integers(0, 10, B)]


def _cpu_lenet_worker(args):
    batch, n_parties, seed = args
    import oracle as O
    from oracle import train_sim as OT
    x, y = lenet_data(batch, seed)

    def step(s):
        m = OT.lenet(s)
        xs = OT.share_fixed(s, x, WIDTH, FRAC, label_key("share:x"))
        ys = OT.share_fixed(s, y, WIDTH, FRAC, label_key("share:y"))
        return m, xs, ys

    dry = O.Sim(n_parties, O.Demand(n_parties))
    m, xs, ys = step(dry)
    m.train_step(dry, xs, ys, LR_SHIFT)
    live = O.Sim(n_parties, O.Store(seed, n_parties, dry.store.demands))
    m, xs, ys = step(live)
    t0 = time.perf_counter()
    m.train_step(live, xs, ys, LR_SHIFT)
    return time.perf_counter() - t0


def cpu_lenet_reference(n_parties: int, cores: int | None = None):
    """The oracle port of the reference algorithm, one LeNet training step of
    batch 128 split data-parallel over all host cores (one process per core,
    batch 128 / cores each; the slowest process bounds the step).
    Fallback when the reference install (baseline/_ref) is missing.
    Returns (steps/s, cores, seconds, per-process batch)."""
    cores = cores or os.cpu_count() or 1
    per = max(1, BATCH // cores)
    procs = -(-BATCH // per)
    ctx = mp.get_context("fork")
    with ctx.Pool(min(cores, procs)) as pool:
        times = pool.map(_cpu_lenet_worker, [(per, n_parties, 11 + i) for i in range(procs)])
    secs = max(times) * (-(-procs // min(cores, procs)))
    return 1.0 / secs, min(cores, procs), secs, per


def reference_arm():
    """baseline/reference_arm.py when the unmodified reference is installed
    in baseline/_ref (it travels to the GPU box with the repo), else None."""
    try:
        from baseline import reference_arm as ra
    except ImportError:
        return None
    return ra if ra.available() is None else None


def ref_train_sampler(ra, arch: str, n_parties: int, batch: int = BATCH, sample: int | None = None):
    """Persistent workers running the reference's online SGD step on the
    batch (or a ``sample`` of it) split over all host cores."""
    cores = os.cpu_count() or 1
    if arch == "lenet":
        x, y = lenet_data(batch)
        keys = (label_key("share:x"), label_key("share:y"))
    else:
        rng = np.random.default_rng(6)
        x, y = rng.uniform(0, 1, (batch, 3, 32, 32)), np.eye(10)[rng.integers(0, 10, batch)]
        keys = ([2, 1], [2, 2])
    if sample is not None:
        x, y = x[:sample], y[:sample]
    procs = min(cores, len(x))
    return ra.TrainWorkers(arch, x, y, n_parties, keys, procs), procs, len(x)


def cpu_baselines(n_parties: int, with_sweep: bool, lenet_steps: int = 2) -> dict:
    """cpu_baseline objects, measured on the host cores before CUDA starts:
    the unmodified reference (kind "reference") when installed, else the
    oracle port (kind "port")."""
    cores = os.cpu_count() or 1
    out = {}
    ra = reference_arm()
    if ra is None:
        sps, c, secs, per = cpu_lenet_reference(n_parties)
        out["lenet"] = {"value": sps, "unit": UNIT, "cores": c, "kind": "port",
                        "sample": f"oracle/ numpy port of the reference algorithm: one LeNet train step of batch "
                                  f"{BATCH} split over {c} processes (batch {per} each, n={n_parties}), online phase, "
                                  f"{secs:.1f} s"}
        if with_sweep:
            rate, rc, rsecs = cpu_reference(1 << 20, 2)
            out["reciprocal"] = {"value": rate, "unit": RECIP_UNIT, "cores": rc, "kind": "port",
                                 "sample": f"online reciprocal on 2^20 elements (n=2), slowest {rsecs:.2f} s"}
        return out
    w, procs, nb = ref_train_sampler(ra, "lenet", n_parties)
    secs = min(w.step() for _ in range(lenet_steps))
    w.close()
    out["lenet"] = {"value": 1.0 / secs, "unit": UNIT, "cores": cores, "kind": "reference",
                    "sample": f"unmodified reference (baseline/_ref): one LeNet SGD step of batch {nb} split over "
                              f"{procs} processes x {n_parties} party threads, online phase {secs:.2f} s"}
    if not with_sweep:
        return out
    chunk = 1 << 13
    for op in ("reciprocal", "exp", "log"):
        tasks = []
        for i in range(cores):
            rng = np.random.default_rng(100 + i)
            xs = workload_inputs(chunk) if op == "reciprocal" else (
                rng.uniform(-16, 16, chunk) if op == "exp" else np.exp2(rng.uniform(-8, 8, chunk)))
            tasks.append(("op", (op, encode_np(xs), 2, label_key(f"share:{op}"))))
        secs = ra.parallel_online(tasks, cores)
        out[op] = {"value": chunk * cores / secs, "unit": RECIP_UNIT, "cores": cores, "kind": "reference",
                   "sample": f"unmodified reference: online {op} on {cores} x 2^13 elements (n=2) at once, "
                             f"slowest {secs:.2f} s"}
    rows, D = 4, 4096
    rng = np.random.default_rng(7)
    b = rng.integers(0, 1 << 64, (D, D), dtype=np.uint64)
    tasks = [("matmul", (rng.integers(0, 1 << 64, (rows, D), dtype=np.uint64), b, 2,
                         (label_key("share:mm_a"), label_key("share:mm_b")))) for _ in range(cores)]
    secs = ra.parallel_online(tasks, cores)
    macs = cores * rows * D * D
    out["matmul"] = {"value": macs / secs / 1e9, "unit": "ring GMAC/s (X@Y, 4096^2 operands)", "cores": cores,
                     "kind": "reference",
                     "sample": f"unmodified reference: online batch_matmul of {cores} x ({rows}x4096 @ 4096x4096) "
                               f"(n=2) at once, slowest {secs:.2f} s"}
    x = np.random.default_rng(3).normal(0, 1, (128, 512))
    secs = ra.parallel_online([("transformer_layer", (x, 2))], 1)
    out["transformer"] = {"value": 6 * secs * 1e3, "unit": "ms (latency, lower is better)", "cores": 2,
                          "kind": "reference",
                          "sample": f"unmodified reference: online forward of 1 of the 6 encoder layers at seq 128 "
                                    f"(n=2, 2 party threads) = {secs:.2f} s, x 6"}
    for arch in ("alexnet", "vgg16m"):
        w, procs, nb = ref_train_sampler(ra, arch, 2, sample=cores)
        secs = w.step()
        w.close()
        out[arch] = {"value": (nb / BATCH) / secs, "unit": UNIT, "cores": cores, "kind": "reference",
                     "sample": f"unmodified reference: online SGD step on {nb} of the {BATCH} images "
                               f"({procs} processes x 2 party threads) = {secs:.2f} s, scaled to batch {BATCH}"}
    return out


# ---------------------------------------------------------------------------
# clocks


class ClockSampler:
    """SM clock + throttle reasons polled every 5 ms from NVML on a host
    thread, so even a ~50 ms timed region holds several samples; falls back
    to `nvidia-smi -lms 50` when NVML is unavailable."""

    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4))

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.thread = None
        self.rows = []
        self.path = tempfile.mktemp(suffix=".csv")

    def _nvml_handle(self):
        import pynvml
        import torch
        pynvml.nvmlInit()
        want = str(getattr(torch.cuda.get_device_properties(self.gpu), "uuid", "")).lower()
        for i in range(pynvml.nvmlDeviceGetCount()):
            h = pynvml.nvmlDeviceGetHandleByIndex(i)
            u = pynvml.nvmlDeviceGetUUID(h)
            u = (u.decode() if isinstance(u, bytes) else str(u)).lower()
            if want and want in u:
                return pynvml, h
        return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.gpu)

    def start(self):
        import threading
        try:
            nv, h = self._nvml_handle()
            self.stop_evt = threading.Event()
            getr = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)

            def poll():
                while not self.stop_evt.is_set():
                    try:
                        self.rows.append((time.time(), float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                                          float(smax), int(getr(h))))
                    except Exception:
                        pass
                    self.stop_evt.wait(0.005)
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.thread = None
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def _smi_rows(self):
        import datetime
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 10:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                mask = sum(bit for (_, bit), v in zip(self.REASONS, parts[6:10]) if v.lower().startswith("active"))
                rows.append((ts, float(parts[2]), float(parts[3]), mask))
            except ValueError:
                continue
        os.unlink(self.path)
        return rows

    def stop(self, window=None) -> dict:
        """Median SM clock and active throttle reasons over the samples taken
        inside ``window`` (host epoch seconds of the timed region)."""
        if self.thread is not None:
            self.stop_evt.set()
            self.thread.join()
            rows, src = self.rows, "nvml 5 ms"
        elif self.proc is not None:
            rows, src = self._smi_rows(), "nvidia-smi 50 ms"
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml / nvidia-smi unavailable"]}
        inside = [r for r in rows if window and window[0] <= r[0] <= window[1]]
        use = inside or rows
        reasons = sorted({nm for r in use for nm, bit in self.REASONS if r[3] & bit})
        return {"sm_mhz": float(np.median([r[1] for r in use])) if use else None,
                "sm_max_mhz": max(r[2] for r in use) if use else None,
                "reasons": reasons, "samples": len(use), "source": src,
                "window": "timed region" if inside else "whole run (no sample fell inside the timed region)"}


# ---------------------------------------------------------------------------
# algorithmic bytes per launch (what the kernel must move)


def alg_bytes(name, a):
    L = None
    try:
        if name == "mpx_carry_fused":
            L, rows, m, s, last = a[7], a[8], a[9], a[10], a[11]
            W = m - s
            rw = W if last else 2 * W
            return L * rows * (16 + (8 if last else 16)) + 3 * L * rows * rw // 8
        if name == "mpx_lmo_fused":
            L, rows, m, s = a[6], a[7], a[8], a[9]
            return L * rows * 16 + 3 * L * rows * (m - s) // 8
        if name == "mpx_mul_fused":
            L, n = a[7], a[8]
            return 6 * L * n * 8
        if name == "mpx_trunc_fused":
            L, n = a[6], a[7]
            return (3 + (1 if a[4] else 0)) * L * n * 8
        if name == "mpx_bit2a_mask":
            L, rows, m = a[5], a[6], a[7]
            return L * rows * 8 + L * rows * m // 8 + rows * 8
        if name == "mpx_bit2a_finish":
            L, rows, m, mode = a[4], a[5], a[6], a[10]
            return rows * 8 + L * rows * m * 8 + (L * rows * m * 8 if mode == 0 else L * rows * 8)
        if name == "mpx_mask_sub":
            L, n = a[4], a[5]
            return 2 * L * n * 8 + n * 8
        if name == "mpx_pubadd_init":
            L, rows, m = a[8], a[9], a[10]
            return rows * 8 + L * rows * m // 8 + 3 * L * rows * 8
        if name == "mpx_sum_from_carries":
            L, rows = a[3], a[4]
            return 3 * L * rows * 8
        if name == "mpx_ring_lin":
            L, n = a[8], a[9]
            return ((1 if a[1] else 0) + (1 if a[3] else 0) + 1) * L * n * 8
        if name == "mpx_bits_op":
            L, rows = a[4], a[5]
            return (2 + (1 if a[2] else 0)) * L * rows * 8
        if name == "mpx_ring_rowdot":
            L, rows, cols = a[3], a[4], a[5]
            return L * rows * cols * 8 + L * rows * 8
        if name == "mpx_bits_gather":
            return 16 * a[4]
        if name == "mpx_gemm_limbs_split":
            # (C, PA8, SA8, PB8, SB8, batch, M, N, Mpad, Npad, Kh, ldc, sC, width, ksplit, Cin, sCin, zl, ...):
            # shared + per-party limb planes read once, the C addend read and Z written (int8 ops: roofline_for)
            batch, M, N, Mpad, Npad, Kh, zl = a[5], a[6], a[7], a[8], a[9], a[10], a[17]
            jobs = batch // max(zl, 1)
            return 8 * Kh * (Mpad + Npad) * (jobs + batch) + (2 if a[15] else 1) * batch * M * N * 8
        if name == "mpx_gemm_limbs":  # int8 ops, not bytes: see roofline_for
            return None
        if name == "mpx_mask_limbs":
            # X_l, T_l read once; shared S limbs + per-party T limbs written
            L, R, Kd, Rpad, Kp = a[10], a[11], a[12], a[13], a[14]
            jobs = a[18] if len(a) > 18 else 1
            return jobs * (2 * L * R * Kd * 8 + (1 + L) * 8 * Rpad * Kp)
        if name == "mpx_mask_limbs2":
            # both sides: X_l, A_l / Y_l, B_l read once; shared + per-party limb planes written
            M, Mpad, N, Npad, L, Kd, Kp, jobs = a[10], a[11], a[22], a[23], a[24], a[25], a[26], a[29]
            return jobs * (2 * L * (M + N) * Kd * 8 + (1 + L) * 8 * (Mpad + Npad) * Kp)
        if name in ("mpx_beaver_gemm", "mpx_beaver_gemm_batched"):
            # D, E read once, A_l, B_l, C_l read and Z_l written per party
            if name == "mpx_beaver_gemm":
                L, batch, M, Kd, N = a[10], 1, a[11], a[12], a[13]
            else:
                L, batch, M, Kd, N = a[14], a[15], a[16], a[17], a[18]
            return 8 * batch * ((1 + L) * (M * Kd + Kd * N) + 2 * L * M * N)
        if name == "mpx_beaver_gemm_sim":
            # X_l, A_l, Y_l, B_l, C_l read once and Z_l written, per party
            L, batch, M, Kd, N = a[22], a[23], a[24], a[25], a[26]
            return 8 * batch * L * (2 * M * Kd + 2 * Kd * N + 2 * M * N)
        if name == "mpx_mask_sub_bs":
            L, batch, n = a[7], a[8], a[9]
            return batch * n * 8 * (2 * L + 1)
        if name == "mpx_mask_sub_t":
            L, batch, rows, cols = a[7], a[8], a[9], a[10]
            return batch * rows * cols * 8 * (2 * L + 1)
        if name == "mpx_beaver_limbs":
            L, M, Kd, N, Mpad, Npad, Kpad = a[8], a[9], a[10], a[11], a[12], a[13], a[14]
            return (1 + L) * 8 * (M * Kd + Kd * N) + L * 8 * (Mpad + Npad) * Kpad
        if name in ("mpx_reciprocal_fused", "mpx_exp_fused", "mpx_log_fused", "mpx_relu_fused",
                    "mpx_maxlevel_fused"):
            from paper_2402_02320_b200.fused import material_bytes
            kind, n, L, calls, io = a
            return material_bytes(calls, L) + io * 8 * L * n   # material + share words in / out
        if name == "mpx_ring_colsum":
            L, rows, cols = a[2], a[3], a[4]
            return 8 * L * rows * cols + 8 * L * cols
        if name in ("mpx_ring_pool_sum", "mpx_ring_pool_scatter"):
            planes, H, W, k, st = a[2], a[3], a[4], a[5], a[6]
            return 8 * planes * H * W + 8 * planes * ((H - k) // st + 1) * ((W - k) // st + 1)
        if name == "mpx_ring_add_rowvec":
            L, rows, cols = a[2], a[3], a[4]
            return 16 * L * rows * cols + 8 * L * cols
        if name == "mpx_im2col":
            L, B, C, H, W, K, st, pd = a[2:10]
            OH, OW = (H + 2 * pd - K) // st + 1, (W + 2 * pd - K) // st + 1
            return 8 * L * B * C * H * W + 8 * L * B * OH * OW * C * K * K
        if name == "mpx_col2im":
            L, B, C, H, W, K, st, pd = a[2:10]
            OH, OW = (H + 2 * pd - K) // st + 1, (W + 2 * pd - K) // st + 1
            return 8 * L * B * C * H * W + 8 * L * B * OH * OW * C * K * K
    except (IndexError, TypeError):
        return None
    return None


INT8_SPEC_TOPS = 4500.0   # B200 nominal dense int8 (B200_PROFILING.md / the task's nominal peaks)


def int8_alt_peak():
    """Second int8 denominator: 2 x the driver-measured bf16 burst."""
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return 2.0 * float(json.load(fh)["bf16_tflops"])
    except (OSError, KeyError, ValueError):
        return None


def _read_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# cfg-5 sweep entries (secondary): Exp / Log on 2^24, Beaver matmul 4096^2


def int8_peak_tops(torch, n=8192, iters=10):
    """cuBLASLt int8 GEMM (torch._int_mm) burst rate: the tensor-pipe roofline
    denominator for int8 (MEASURED_PEAKS.json only carries bf16)."""
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = None
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return 2 * n ** 3 / (best / 1e3) / 1e12


def philox_ceiling_gblocks(torch, blocks=1 << 28, iters=5):
    """Philox4x64-10 ALU ceiling (mpx_philox_probe: generate + XOR-fold, no
    stores), G blocks/s, best of `iters`: the dealer's roofline denominator."""
    from paper_2402_02320_b200 import kernels as K
    out = torch.empty(148 * 8 * 256, dtype=torch.int64, device="cuda")
    K.philox_probe(out, 1 << 20)
    torch.cuda.synchronize()
    best = None
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        K.philox_probe(out, blocks)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return blocks / (best / 1e3) / 1e9


def dealer_roofline(torch, demands, n_parties, needs_bits, dealer_ms):
    """The re-deal's Philox work (preprocessing.stream_blocks: every draw of
    the reference's generate_material, 32 bytes per block) over its time,
    against the in-run ALU ceiling."""
    from paper_2402_02320_b200.preprocessing import stream_blocks
    blocks = stream_blocks(demands, n_parties, needs_bits)
    peak = philox_ceiling_gblocks(torch)
    achieved = blocks / (dealer_ms / 1e3) / 1e9
    return {"bound": "alu (Philox4x64-10)", "achieved": achieved, "peak": peak, "unit": "G Philox blocks/s",
            "frac": achieved / peak, "blocks_per_deal": blocks,
            "peak_kind": "measured in-run: mpx_philox_probe (Philox4x64-10 generate + XOR-fold, no stores)",
            "note": "whole re-deal incl. the matrix-triple C = A @ B GEMMs and all share stores"}


def sweep_entry(torch, G, make_session, parties, n_parties, dev, name, steps=2, warmup=1, elems=1 << 24):
    from paper_2402_02320_b200 import _lib
    from paper_2402_02320_b200.preprocessing import DemandCounter, device_store
    from paper_2402_02320_b200.protocols import batch_matmul
    N = elems
    rng = np.random.default_rng(7)
    if name == "matmul":
        D = 4096
        a = rng.integers(0, 1 << 64, (D, D), dtype=np.uint64)
        b = rng.integers(0, 1 << 64, (D, D), dtype=np.uint64)

        def inputs(s):
            return s.share_ring(a, 64, 0, label_key("share:mm_a")), s.share_ring(b, 64, 0, label_key("share:mm_b"))

        def op(s, x, y):
            return batch_matmul(s, [(x, y)])[0]
    else:
        xs = rng.uniform(-16, 16, N) if name == "exp" else np.exp2(rng.uniform(-8, 8, N))
        enc = encode_np(xs)

        def inputs(s):
            x = s.share_ring(enc, WIDTH, FRAC, label_key(f"share:{name}"))
            return x, None

        def op(s, x, y):
            return G.exponentiation(s, x) if name == "exp" else G.logarithm(s, x)
    counter = DemandCounter(parties, n_parties)
    sd = make_session(counter)
    op(sd, *inputs(sd))
    x, y = inputs(make_session(None))
    times, prof_ms = [], {}
    store = None
    for step in range(warmup + steps):
        del store
        store = device_store(500 + step, n_parties, counter.demands, parties=parties, device=dev,
                             needs_bits=counter.needs_bits)
        sess = make_session(store)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if step == warmup + steps - 1:
            _lib.profile_begin()
        e0.record()
        op(sess, x, y)
        e1.record()
        torch.cuda.synchronize()
        if _lib.profiling() is not None:
            prof = _lib.profile_end()
            for nm, _a, p0, p1 in prof:
                prof_ms[nm] = prof_ms.get(nm, 0.0) + p0.elapsed_time(p1)
            per = _profile_kernels(prof)
        if step >= warmup:
            times.append(e0.elapsed_time(e1))
    del store
    ms = float(np.mean(times))
    out = {"ms_per_op": ms, "steps": steps}
    if name != "matmul":
        out["roofline"] = roofline_for(per)
    if name == "matmul":
        macs = len(parties) * D * (2 * D) * D          # [D|A_l] @ [B_l';E] per local party
        tc_ms = prof_ms.get("mpx_gemm_limbs", 0.0) + prof_ms.get("mpx_gemm_limbs_split", 0.0)
        out.update({"shape": [D, D, D], "ring_GMAC_per_s": macs / (ms / 1e3) / 1e9,
                    "gemm_kernel_ms": tc_ms,
                    "gemm_int8_TOPS": 36 * 2 * macs / (tc_ms / 1e3) / 1e12 if tc_ms else None})
    else:
        out.update({"elements": N, "elements_per_s": N / (ms / 1e3)})
    return out


# ---------------------------------------------------------------------------
# B200 arm


class DistGroup:
    """torch.distributed over NCCL: one rank per GPU (torchrun)."""

    capturable = True   # NCCL collectives can be captured into the step's CUDA graph

    def __init__(self, torch, dist):
        self.torch, self.dist = torch, dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))

    def init(self, dev):
        if self.world > 1:
            # communicator init lines on stderr (one per rank) show the N-rank NCCL setup
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            self.dist.init_process_group("nccl", device_id=dev)

    def comm(self):
        return None            # PartySession default: DistComm over the NCCL group

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, v: float, dev) -> float:
        if self.world == 1:
            return v
        t = self.torch.tensor([v], device=dev, dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def _profile_kernels(prof):
    per = {}
    for name, a, e0, e1 in prof:
        d = per.setdefault(name, {"ms": 0.0, "n": 0, "bytes": 0, "bytes_known": True, "ops": 0})
        d["ms"] += e0.elapsed_time(e1)
        d["n"] += 1
        if name == "mpx_gemm_limbs":
            # (C, A8, B8, batch, M, N, Mpad, Npad, Kpad, ...): 36 limb MACs per ring MAC
            d["ops"] += 2 * 36 * a[3] * a[4] * a[5] * a[8]
        elif name == "mpx_gemm_limbs_split":
            # (C, PA8, SA8, PB8, SB8, batch, M, N, Mpad, Npad, Kh, ...): reduction length 2 Kh
            d["ops"] += 2 * 36 * a[5] * a[6] * a[7] * 2 * a[10]
        b = alg_bytes(name, a)
        if b is None:
            d["bytes_known"] = False
        else:
            d["bytes"] += b
    return per


def roofline_for(per, int8_peak=None):
    """Roofline object of the dominant kernel of one profiled step."""
    step_ms = sum(d["ms"] for d in per.values())
    dom_name = max(per, key=lambda k: per[k]["ms"])
    dom = per[dom_name]
    common = {"kernel": dom_name, "launches": dom["n"], "avg_launch_us": 1e3 * dom["ms"] / dom["n"],
              "share_of_step": dom["ms"] / step_ms}
    traffic = None
    tpath = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(dom_name)
        except ValueError:
            traffic = None
    if dom_name in ("mpx_gemm_limbs", "mpx_gemm_limbs_split"):
        ach = dom["ops"] / (dom["ms"] / 1e3) / 1e12
        alt = int8_alt_peak()
        hbm_peak, _ = _read_peaks()
        hbm = (dom["bytes"] / (dom["ms"] / 1e3) / 1e9) if dom["bytes_known"] and dom["bytes"] else None
        return dict(common, bound="tensor", achieved=ach, peak=int8_peak, unit="TOPS int8",
                    hbm_view={"achieved_GBps": hbm, "peak_GBps": hbm_peak,
                              "frac": (hbm / hbm_peak) if hbm else None,
                              "alg_bytes_per_launch": (dom["bytes"] // dom["n"]) if hbm else None,
                              "note": "limb planes read once + C addend read + Z written: the thin LeNet "
                                      "products are operand/epilogue paced, so both views are reported"},
                    peak_kind="measured in-run: torch._int_mm int8 8192^3 (cuBLASLt), burst "
                              "(MEASURED_PEAKS.json carries bf16 only)",
                    frac=(ach / int8_peak) if int8_peak else None, traffic=traffic,
                    peak_alt=alt, frac_alt=(ach / alt) if alt else None,
                    peak_alt_kind="2 x MEASURED_PEAKS.json bf16_tflops (dense int8 = 2x bf16 on B200)",
                    peak_spec=INT8_SPEC_TOPS, frac_spec=ach / INT8_SPEC_TOPS,
                    traffic_unit="DRAM bytes per launch (ncu)", alg_ops_per_launch=dom["ops"] // dom["n"])
    peak, peak_kind = _read_peaks()
    ach = dom["bytes"] / (dom["ms"] / 1e3) / 1e9 if dom["bytes_known"] else None
    return dict(common, bound="hbm", achieved=ach, peak=peak, peak_kind=peak_kind, unit="GB/s",
                frac=(ach / peak) if ach else None, traffic=traffic,
                alg_bytes_per_launch=dom["bytes"] // dom["n"])


def _kernel_table(per):
    return {k: {"ms": round(v["ms"], 3), "launches": v["n"],
                "GBps": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 1) if v["bytes_known"] and v["ms"] else None}
            for k, v in sorted(per.items(), key=lambda kv: -kv[1]["ms"])}


def reciprocal_entry(torch, G, make_session, parties, n_parties, dev, group, steps, warmup, elems=1 << 24):
    """cfg 5: secure Reciprocal on 2^24 elements (one fused kernel in sim mode)."""
    from paper_2402_02320_b200 import _lib
    from paper_2402_02320_b200.preprocessing import DemandCounter, device_store
    N = elems
    xs = workload_inputs(N)
    enc = encode_np(xs)
    key = label_key("share:x")
    counter = DemandCounter(parties, n_parties)
    sd = make_session(counter)
    G.reciprocal(sd, sd.share_ring(enc, WIDTH, FRAC, key))
    x_sh = make_session(None).share_ring(enc, WIDTH, FRAC, key)
    times, store = [], None
    for step in range(warmup + steps + 1):
        del store
        store = device_store(3000 + step, n_parties, counter.demands, parties=parties, device=dev,
                             needs_bits=counter.needs_bits)
        sess = make_session(store)
        group.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        last = step == warmup + steps
        if last:
            _lib.profile_begin()
        e0.record()
        y = G.reciprocal(sess, x_sh)
        e1.record()
        torch.cuda.synchronize()
        if last:
            per = _profile_kernels(_lib.profile_end())
        elif step >= warmup:
            times.append(e0.elapsed_time(e1))
    ms = group.max(float(np.mean(times)), dev)
    y_open = sess.open_fixed(y)
    xq = enc.view(np.int64) / float(1 << FRAC)
    del store
    return {"elements": N, "ms_per_op": ms, "elements_per_s": N / (ms / 1e3), "steps": steps,
            "max_rel_err": float(np.max(np.abs(y_open - 1 / xq) * np.abs(xq))),
            "roofline": roofline_for(per), "kernels": _kernel_table(per)}


def mlp_entry(torch, dev, steps, warmup):
    """configs[0]: 2-party Simple MLP (784-128-128-10) forward+backward+SGD, batch 128."""
    from paper_2402_02320_b200 import train
    from paper_2402_02320_b200.preprocessing import DemandCounter, device_store
    from paper_2402_02320_b200.session import SimSession
    n = 2
    rng = np.random.default_rng(5)
    x, y = rng.normal(0, 1, (BATCH, 784)), np.eye(10)[rng.integers(0, 10, BATCH)]
    c = DemandCounter((0, 1), n)
    sd = SimSession(n, c, device=dev)
    train.simple_mlp(sd).train_step(sd, sd.share_fixed(x, WIDTH, FRAC, [1, 1]), sd.share_fixed(y, WIDTH, FRAC, [1, 2]),
                                    LR_SHIFT)
    s = SimSession(n, None, device=dev)
    m = train.simple_mlp(s)
    g = train.GraphedStep(s, m, s.share_fixed(x, WIDTH, FRAC, [1, 1]), s.share_fixed(y, WIDTH, FRAC, [1, 2]),
                          LR_SHIFT, c.demands, c.needs_bits, seed0=70)
    times = []
    for t in range(warmup + steps):
        g.dealer.redeal(71 + t)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.graph.replay()
        e1.record()
        torch.cuda.synchronize()
        if t >= warmup:
            times.append(e0.elapsed_time(e1))
    ms = float(np.mean(times))
    return {"model": "Simple MLP 784-128-128-10", "parties": n, "batch": BATCH, "ms_per_step": ms,
            "steps_per_s": 1e3 / ms, "cuda_graph": True}


def cifar_entry(torch, dev, arch, steps, warmup, n=2):
    """configs[2]: AlexNet / VGG16m training step (paper tables) on a synthetic
    CIFAR-10-shape batch of 128, n parties simulated on one GPU, CUDA graph."""
    from paper_2402_02320_b200 import train
    from paper_2402_02320_b200.preprocessing import DemandCounter, device_store
    from paper_2402_02320_b200.session import SimSession
    rng = np.random.default_rng(6)
    shape = (BATCH, 1, 28, 28) if arch == "lenet" else (BATCH, 3, 32, 32)
    x, y = rng.uniform(0, 1, shape), np.eye(10)[rng.integers(0, 10, BATCH)]
    build = getattr(train, arch)
    c = DemandCounter(tuple(range(n)), n)
    sd = SimSession(n, c, device=dev)
    md = build(sd)
    p = md.layers[0].p
    md.train_step(sd, sd.share_fixed(x, WIDTH, p, [2, 1]), sd.share_fixed(y, WIDTH, p, [2, 2]), LR_SHIFT)
    s = SimSession(n, None, device=dev)
    m = build(s)
    g = train.GraphedStep(s, m, s.share_fixed(x, WIDTH, p, [2, 1]), s.share_fixed(y, WIDTH, p, [2, 2]),
                          LR_SHIFT, c.demands, c.needs_bits, seed0=80)
    times, deal = [], []
    for t in range(warmup + steps):
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record()
        g.dealer.redeal(81 + t)
        d1.record()
        torch.cuda.synchronize()
        deal.append(d0.elapsed_time(d1))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.graph.replay()
        e1.record()
        torch.cuda.synchronize()
        if t >= warmup:
            times.append(e0.elapsed_time(e1))
    ms = float(np.mean(times))
    mat = sum(t.numel() * t.element_size() for d in s.store._arrays.values() for t in d.values())
    return {"model": arch, "params": m.n_params, "parties": n, "batch": BATCH, "frac": p, "ms_per_step": ms,
            "steps_per_s": 1e3 / ms, "rounds_per_step": sd.metrics.total.rounds,
            "material_GB_per_step": mat / 1e9, "dealer_ms_per_step": float(np.median(deal[warmup:])),
            "cuda_graph": True}


def transformer_entry(torch, dev, steps, warmup, n=2):
    """configs[3]: 18.9M-parameter Transformer secure inference, seq 128, p = 14,
    2 parties on one GPU, forward captured in one CUDA graph. Latency per
    forward (lower is better)."""
    from paper_2402_02320_b200.preprocessing import DemandCounter, device_store
    from paper_2402_02320_b200.session import SimSession
    from paper_2402_02320_b200.transformer import GraphedInference, Transformer
    S = 128
    x = np.random.default_rng(3).normal(0, 1, (S, 512))
    c = DemandCounter(tuple(range(n)), n)
    sd = SimSession(n, c, device=dev)
    Transformer(sd).forward(sd, sd.share_fixed(x, WIDTH, 14, [5, 5]))
    s = SimSession(n, None, device=dev)
    m = Transformer(s)
    g = GraphedInference(s, m, s.share_fixed(x, WIDTH, 14, [5, 5]), c.demands, c.needs_bits, seed0=90)
    times = []
    for t in range(warmup + steps):
        g.dealer.redeal(91 + t)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.graph.replay()
        e1.record()
        torch.cuda.synchronize()
        if t >= warmup:
            times.append(e0.elapsed_time(e1))
    y = s.open_fixed(g.y)
    xq = np.floor(x * (1 << 14)) / (1 << 14)
    return {"model": "6-layer encoder d512 h8 ffn2048 (18,874,368 secret weights)", "seq": S, "parties": n,
            "frac": 14, "latency_ms": float(np.mean(times)), "higher_is_better": False,
            "rounds": sd.metrics.total.rounds, "cuda_graph": True,
            "max_abs_err_vs_float64": float(np.abs(y - m.plaintext(xq)).max())}


def party_mode_entry(torch, dev, n: int = 3, steps: int = 5, warmup: int = 2):
    """The one-party-per-GPU (L = 1) LeNet step of party 0 on this GPU with
    the collectives elided (session.LoopbackComm): the per-party compute of
    the north star's n-GPU deployment, captured in a CUDA graph like the sim
    step, plus what the n-GPU run adds on top - the rounds and the bytes this
    party's collectives move per step (all_reduce for arithmetic openings,
    all_gather + XOR kernel for bit openings)."""
    from paper_2402_02320_b200 import train
    from paper_2402_02320_b200.preprocessing import DemandCounter
    from paper_2402_02320_b200.session import LoopbackComm, PartySession
    x, y = lenet_data(BATCH)
    kx, ky = label_key("share:x"), label_key("share:y")
    c = DemandCounter((0,), n)
    sd = PartySession(0, n, LoopbackComm(n), c, device=dev)
    train.lenet(sd).train_step(sd, sd.share_fixed(x, WIDTH, FRAC, kx), sd.share_fixed(y, WIDTH, FRAC, ky), LR_SHIFT)
    s = PartySession(0, n, LoopbackComm(n), None, device=dev)
    m = train.lenet(s)
    before = s.metrics.physical_bytes
    g = train.GraphedStep(s, m, s.share_fixed(x, WIDTH, FRAC, kx), s.share_fixed(y, WIDTH, FRAC, ky), LR_SHIFT,
                          c.demands, c.needs_bits, seed0=300)
    phys = (s.metrics.physical_bytes - before) // 2           # warm-up step + captured step
    times = []
    for t in range(warmup + steps):
        g.dealer.redeal(301 + t)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.graph.replay()
        e1.record()
        torch.cuda.synchronize()
        if t >= warmup:
            times.append(e0.elapsed_time(e1))
    tot = sd.metrics.total.as_dict()
    return {"parties": n, "party": 0, "batch": BATCH, "local_compute_ms_per_step": float(np.mean(times)),
            "rounds_per_step": tot["rounds"], "logical_bytes_sent_per_step": tot["bytes"],
            "collective_bytes_per_step": int(phys),
            "how": "PartySession(L=1) of party 0 with LoopbackComm (collectives elided), CUDA graph replay; "
                   "an n-GPU run adds one NCCL collective per round on top"}


def party_scaling(torch, G, dev, group, ns=(2, 4, 8)):
    """North-star party sweep, all n parties simulated on one GPU (one-GPU-
    per-party runs need an n-GPU box: bench.py --gpus n under torchrun):
    LeNet / AlexNet / VGG16m training steps (configs[1], configs[2]), 18.9M
    Transformer inference, Beaver matmul 4096^2,
    and Reciprocal / Exp / Log on 2^22 elements (2^24 x 8 parties of
    single-use material would exceed HBM)."""
    from paper_2402_02320_b200.session import SimSession
    out = {}
    for n in ns:
        def mk(store, n=n):
            return SimSession(n, store, device=dev)
        parties = tuple(range(n))
        e = {"lenet_train_ms": cifar_entry(torch, dev, "lenet", 3, 2, n=n)["ms_per_step"],
             "transformer_infer_ms": transformer_entry(torch, dev, 3, 2, n=n)["latency_ms"]}
        # configs[2] at 2/4/8 parties: AlexNet, and VGG16m where its single-use
        # material (~15 GB per party per step) still fits HBM next to the step
        for arch in ("alexnet", "vgg16m"):
            try:
                ce = cifar_entry(torch, dev, arch, 2, 1, n=n)
                e[f"{arch}_train_ms"] = ce["ms_per_step"]
                e[f"{arch}_material_GB"] = ce["material_GB_per_step"]
            except torch.cuda.OutOfMemoryError as err:
                e[f"{arch}_train_ms"] = None
                e[f"{arch}_skipped"] = f"out of device memory at n = {n} ({str(err).splitlines()[0][:120]})"
            torch.cuda.empty_cache()
        mm = sweep_entry(torch, G, mk, parties, n, dev, "matmul")
        e["matmul_4096_ms"] = mm["ms_per_op"]
        r = reciprocal_entry(torch, G, mk, parties, n, dev, group, 2, 1, elems=1 << 22)
        e["reciprocal_2^22_ms"] = r["ms_per_op"]
        e["reciprocal_hbm_frac"] = r["roofline"]["frac"]
        for nm in ("exp", "log"):
            s = sweep_entry(torch, G, mk, parties, n, dev, nm, elems=1 << 22)
            e[f"{nm}_2^22_ms"] = s["ms_per_op"]
            e[f"{nm}_hbm_frac"] = s["roofline"]["frac"]
        out[str(n)] = e
    return out


def run_b200(args, group=None):
    import torch
    import torch.distributed as dist

    import paper_2402_02320_b200 as G
    from paper_2402_02320_b200 import _lib, train
    from paper_2402_02320_b200.preprocessing import DemandCounter, device_store
    from paper_2402_02320_b200.session import PartySession, SimSession

    group = group or DistGroup(torch, dist)
    world, rank, local = group.world, group.rank, group.local
    n_parties = 3 if world == 1 else world
    cpu_all = {}
    if rank == 0 and world == 1 and not args.no_cpu:
        # before CUDA initialisation: the pools fork numpy-only workers
        cpu_all = cpu_baselines(n_parties, with_sweep=not args.no_sweep)
    cpu = cpu_all.get("lenet")
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group.init(dev)
    parties = tuple(range(n_parties)) if world == 1 else (rank,)

    def make_session(store):
        if world == 1:
            return SimSession(n_parties, store, device=dev)
        return PartySession(rank, n_parties, group.comm(), store, device=dev)

    B = args.batch
    x, y = lenet_data(B)
    kx, ky = label_key("share:x"), label_key("share:y")
    # dry run: exact demand of one training step
    counter = DemandCounter(parties, n_parties)
    sd = make_session(counter)
    train.lenet(sd).train_step(sd, sd.share_fixed(x, WIDTH, FRAC, kx), sd.share_fixed(y, WIDTH, FRAC, ky), LR_SHIFT)
    sess = make_session(None)
    model = train.lenet(sess)
    xs, ys = sess.share_fixed(x, WIDTH, FRAC, kx), sess.share_fixed(y, WIDTH, FRAC, ky)
    launches_per_step = None
    graph = None
    graph_note = None
    l0 = _lib.LAUNCHES
    try:
        if world > 1 and not getattr(group, "capturable", False):
            raise RuntimeError("the party group's collectives are host rendezvous (not capturable)")
        # party mode (N > 1): the NCCL collectives of every round are captured
        # into the step's CUDA graph too (thread-local capture: the NCCL
        # watchdog thread keeps polling its own events)
        graph = train.GraphedStep(sess, model, xs, ys, LR_SHIFT, counter.demands, counter.needs_bits, seed0=1,
                                  capture_error_mode="global" if world == 1 else "thread_local")
        launches_per_step = (_lib.LAUNCHES - l0) // 2          # warm-up step + captured step
    except Exception as e:  # noqa: BLE001
        if world == 1:
            raise
        graph_note = f"CUDA-graph capture of the NCCL step failed ({type(e).__name__}: {e}); eager steps"
        print(f"[rank {rank}] {graph_note}", file=sys.stderr)
        torch.cuda.synchronize(dev)
        graph = None
        sess.store = device_store(1, n_parties, counter.demands, parties=parties, device=dev,
                                  needs_bits=counter.needs_bits)

    def redeal(seed):
        if graph is not None:          # the dealer's own CUDA graph (DealerGraph)
            graph.dealer.redeal(seed)
        else:
            device_store(seed, n_parties, counter.demands, parties=parties, device=dev,
                         needs_bits=counter.needs_bits, into=sess.store)

    def one_step():
        if graph is not None:
            graph.graph.replay()
            return graph.logits
        return model.train_step(sess, xs, ys, LR_SHIFT)

    losses = []

    def loss_of(logits, yy):
        z = sess.open_fixed(logits)
        z = z - z.max(1, keepdims=True)
        p = np.exp(z) / np.exp(z).sum(1, keepdims=True)
        return float(-np.mean(np.log(p[np.arange(len(yy)), yy.argmax(1)] + 1e-12)))

    clocks = ClockSampler(local)
    clocks.start()
    step_ms, deal_ms, t_window = [], [], [None, None]
    for step in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record()
        redeal(100 + step)
        d1.record()
        torch.cuda.synchronize()
        deal_ms.append((d0.elapsed_time(d1), 1e3 * (time.perf_counter() - t0)))
        group.barrier()
        torch.cuda.synchronize()
        if step >= args.warmup and t_window[0] is None:
            t_window[0] = time.time()
        l0 = _lib.LAUNCHES
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        logits = one_step()
        e1.record()
        torch.cuda.synchronize()
        group.barrier()
        if launches_per_step is None:
            launches_per_step = _lib.LAUNCHES - l0
        if step >= args.warmup:
            step_ms.append(e0.elapsed_time(e1))
            t_window[1] = time.time()
        if step in (0, args.warmup + args.steps - 1):
            losses.append(loss_of(logits, y))
    clk = clocks.stop(t_window)
    total_ms = group.max(float(sum(step_ms)), dev)
    value = args.steps / (total_ms / 1e3)

    # profiled eager step (per-kernel CUDA events): dominant kernel + roofline
    redeal(9000)
    torch.cuda.synchronize()
    _lib.profile_begin()
    model.train_step(sess, xs, ys, LR_SHIFT)
    torch.cuda.synchronize()
    per = _profile_kernels(_lib.profile_end())
    if graph is not None:
        graph._writeback()
    int8_pk = int8_peak_tops(torch) if world == 1 else None
    roofline = roofline_for(per, int8_pk)

    # e2e through the public API with host buffers: H2D of the step's input
    # shares into the step's (static) input tensors, the step, D2H of the logits
    x_host = xs.values.cpu().pin_memory()
    y_host = ys.values.cpu().pin_memory()
    out_host = None
    e2e = []
    for step in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        redeal(20_000 + step)
        group.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        xs.values.copy_(x_host, non_blocking=True)
        ys.values.copy_(y_host, non_blocking=True)
        logits = one_step()
        if out_host is None:
            out_host = torch.empty(logits.values.shape, dtype=torch.int64).pin_memory()
        out_host.copy_(logits.values, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        group.barrier()
        if step >= args.warmup:
            e2e.append(e0.elapsed_time(e1))
    e2e_total = group.max(float(sum(e2e)), dev)

    sweep = {}
    if not args.no_sweep:
        ps = (0, 1) if world == 1 else parties
        np_ = 2 if world == 1 else n_parties

        def mk2(store):
            if world == 1:
                return SimSession(2, store, device=dev)
            return PartySession(rank, n_parties, group.comm(), store, device=dev)
        sweep["reciprocal"] = reciprocal_entry(torch, G, mk2, ps, np_, dev, group, 3, 2)
        for nm in ("exp", "log", "matmul"):
            sweep[nm] = sweep_entry(torch, G, mk2, ps, np_, dev, nm)
        if int8_pk:
            mm = sweep["matmul"]
            mm["roofline"] = {"bound": "tensor", "kernel": "mpx_gemm_limbs (tcgen05 kind::i8)",
                              "achieved": mm.get("gemm_int8_TOPS"), "peak": int8_pk,
                              "peak_kind": "measured in-run: torch._int_mm int8 8192^3 (cuBLASLt), burst",
                              "unit": "TOPS int8",
                              "frac": (mm["gemm_int8_TOPS"] / int8_pk) if mm.get("gemm_int8_TOPS") else None,
                              "peak_alt": int8_alt_peak(), "peak_spec": INT8_SPEC_TOPS,
                              "frac_spec": (mm["gemm_int8_TOPS"] / INT8_SPEC_TOPS) if mm.get("gemm_int8_TOPS") else None,
                              "frac_alt": (mm["gemm_int8_TOPS"] / int8_alt_peak())
                              if mm.get("gemm_int8_TOPS") and int8_alt_peak() else None}
        if world == 1:
            sweep["mlp_train"] = mlp_entry(torch, dev, 5, 3)
            sweep["transformer"] = transformer_entry(torch, dev, 3, 2)
            for arch in ("alexnet", "vgg16m"):
                sweep[f"{arch}_train"] = cifar_entry(torch, dev, arch, 3, 2)
            sweep["party_mode_1gpu"] = {str(n): party_mode_entry(torch, dev, n) for n in (2, 3, 4, 8)}
            if not getattr(args, "no_party_sweep", False):
                sweep["party_scaling_sim"] = party_scaling(torch, G, dev, group)
        for nm, key in (("reciprocal", "reciprocal"), ("exp", "exp"), ("log", "log"), ("matmul", "matmul"),
                        ("transformer", "transformer"), ("alexnet_train", "alexnet"), ("vgg16m_train", "vgg16m")):
            if nm in sweep:
                sweep[nm]["cpu_baseline"] = cpu_all.get(key)

    line = None
    dealer_roof = None
    if rank == 0:
        if world == 1:   # all parties' draws on this GPU (party mode deals one party's share of the work)
            dealer_roof = dealer_roofline(torch, counter.demands, n_parties, counter.needs_bits,
                                          float(np.median([d[0] for d in deal_ms[args.warmup:]])))
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64 (Z_2^64 fixed point, p=23)",
            "data": "synthetic: x ~ U(0,1) 128x1x28x28, uniform labels; Kaiming-init secret weights",
            "config": {"workload": LENET_WORKLOAD,
                       "parties": n_parties, "batch": B, "frac": FRAC, "ring_width": WIDTH,
                       "mode": ("sim: all parties on 1 GPU, step captured in one CUDA graph" if world == 1
                                else "one party per GPU, NCCL openings" +
                                (", step (kernels + collectives) captured in one CUDA graph" if graph is not None
                                 else ", eager (" + str(graph_note) + ")")),
                       "l2": "working set > L2 per step (material ~1.4 GB, re-dealt in place each step)",
                       "dealer": "fresh on-device material re-dealt in place before every step, outside "
                                 "the timed region"},
            "e2e": {"value": args.steps / (e2e_total / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": int(x_host.numel() * 8 + y_host.numel() * 8),
                    "d2h_bytes_per_step": int(out_host.numel() * 8), "ms_per_step": e2e_total / args.steps,
                    "how": "pinned host input shares -> step input tensors (H2D), the train step, logits "
                           "shares -> pinned host (D2H), all inside the CUDA-event window"},
            "gpu_launches": launches_per_step * args.steps,
            "gpu_launches_per_step": launches_per_step,
            "clocks": clk,
            "roofline": roofline,
            "rounds_per_step": sd.metrics.total.rounds,
            "dealer_ms_per_step": float(np.median([d[0] for d in deal_ms[args.warmup:]])),
            "dealer": {"gpu_ms_per_step": float(np.median([d[0] for d in deal_ms[args.warmup:]])),
                       "host_wall_ms_per_step": float(np.median([d[1] for d in deal_ms[args.warmup:]])),
                       "how": ("one CUDA graph of the whole re-deal (keys in device slots), CUDA events"
                               if world == 1 else "device_store(into=...) per step, CUDA events"),
                       "material_GB": sum(t.numel() * t.element_size() for d in sess.store._arrays.values()
                                          for t in d.values()) / 1e9,
                       "roofline": dealer_roof},
            "loss_first_last": losses,
            "kernels": _kernel_table(per),
            "cpu_baseline": cpu,
            "sweep": sweep,
        }
    group.close()
    return line


def run_reference(args):
    """The reference arm: the unmodified reference (baseline/_ref) on all host
    cores, same metric / config / unit as the B200 arm; each step = one online
    LeNet SGD step of batch 128 split over the cores (dry run + dealer once
    per worker, outside the timed region). Falls back to the oracle port when
    the reference install is missing."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_parties = 3 if world == 1 else world
    ra = reference_arm()
    rates = []
    if ra is not None:
        w, procs, nb = ref_train_sampler(ra, "lenet", n_parties)
        for step in range(args.warmup + args.steps):
            secs = w.step()
            if step >= args.warmup:
                rates.append(1.0 / secs)
        w.close()
        cores = os.cpu_count() or 1
        kind, mode = "reference", "CPU: unmodified reference package (baseline/_ref), all host cores"
        sample = (f"each step: batch {nb} split over {procs} processes x {n_parties} party threads (InProcHub), "
                  f"online phase; dry run + reference dealer once per process")
    else:
        cores = per = None
        for step in range(args.warmup + args.steps):
            sps, cores, secs, per = cpu_lenet_reference(n_parties)
            if step >= args.warmup:
                rates.append(sps)
        kind, mode = "port", "CPU: reference algorithm (numpy oracle port; baseline/_ref missing), all host cores"
        sample = f"each step: batch {BATCH} split over {cores} processes (batch {per} each), online phase"
    value = float(np.mean(rates))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 / value, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64 (Z_2^64 fixed point, p=23)", "impl": "reference",
            "data": "synthetic: x ~ U(0,1) 128x1x28x28, uniform labels; Kaiming-init secret weights",
            "config": {"workload": LENET_WORKLOAD, "parties": n_parties,
                       "batch": BATCH, "frac": FRAC, "ring_width": WIDTH, "mode": mode},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--cpu-sample", type=int, default=1 << 20)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-party-sweep", action="store_true")
    ap.add_argument("--chunks", type=int, default=8)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        line = run_b200(args)
        if line is not None:
            print(json.dumps(line))


if __name__ == "__main__":
    main()
