"""One CUDA engine per device: owns the C-ABI handle, the ln-k table and the draw tables.

PyTorch is used only for device buffers and the current CUDA stream (plumbing).  Every
numeric step of the hot path runs in ``libzks_b200.so``.
"""
from __future__ import annotations

import ctypes
import threading
from collections import OrderedDict

import numpy as np

from . import _native
from .series import natural_logs

_LOG_LEN = 65537  # ln k for k = 0..65536 (tail endpoints reach 65536)


def _torch():
    import torch

    return torch


class DrawTable:
    """A sampling CDF resident on the device plus its guide table (zks_table)."""

    __slots__ = ("handle", "length", "engine")

    def __init__(self, engine: "Engine", cdf: np.ndarray):
        cdf = np.ascontiguousarray(cdf, dtype=np.float64)
        out = ctypes.c_void_p()
        engine.bind_stream()
        _native.check(engine.lib.zks_table_create(engine.handle, cdf.ctypes.data, cdf.size, ctypes.byref(out)))
        self.handle = out
        self.length = int(cdf.size)
        self.engine = engine

    def close(self) -> None:
        if self.handle:
            self.engine.lib.zks_table_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Engine:
    """CUDA engine bound to one device (one per process and device)."""

    def __init__(self, device: int | None = None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("zipfks_b200 needs a CUDA device (sm_100a); none is visible")
        self.lib = _native.load()
        self.device = torch.cuda.current_device() if device is None else int(device)
        logs = np.ascontiguousarray(natural_logs(_LOG_LEN - 1), dtype=np.float64)
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _native.check(self.lib.zks_engine_create(self.device, logs.ctypes.data, logs.size, ctypes.byref(handle)))
        self.handle = handle
        self._tables: OrderedDict[tuple, DrawTable] = OrderedDict()
        self._lock = threading.Lock()
        self.rng = "numpy"

    # -- streams -------------------------------------------------------------
    def bind_stream(self):
        """Enqueue engine work on torch's current stream of this device."""
        torch = _torch()
        stream = torch.cuda.current_stream(self.device)
        _native.check(self.lib.zks_engine_set_stream(self.handle, ctypes.c_void_p(stream.cuda_stream)))
        return stream

    def sync(self) -> None:
        _native.check(self.lib.zks_engine_sync(self.handle))

    @property
    def launches(self) -> int:
        """CUDA kernels this engine has enqueued so far (counted in the native library; bench.py
        reports the timed-region delta)."""
        out = ctypes.c_ulonglong()
        _native.check(self.lib.zks_engine_launches(self.handle, ctypes.byref(out)))
        return out.value

    def set_timing(self, on: bool) -> None:
        """Bracket every kernel launch with CUDA events on the engine stream (diagnostics)."""
        _native.check(self.lib.zks_engine_set_timing(self.handle, int(bool(on))))

    def kernel_times(self) -> dict:
        """{kind: (milliseconds, launches)} since the last call (synchronises; resets)."""
        n = len(_native.KERNEL_KINDS)
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_ulonglong * n)()
        _native.check(self.lib.zks_engine_kernel_times(self.handle, ms, cnt))
        return {k: (ms[i], cnt[i]) for i, k in enumerate(_native.KERNEL_KINDS)}

    # -- tables --------------------------------------------------------------
    def has_table(self, gamma: float, support_k: int | None) -> bool:
        with self._lock:
            return (float(gamma), support_k) in self._tables

    def table(self, gamma: float, support_k: int | None, cdf_builder) -> DrawTable:
        """Cached device table for the generating model (montecarlo.py:82-86 lru_cache)."""
        key = (float(gamma), support_k)
        with self._lock:
            t = self._tables.get(key)
            if t is not None:
                self._tables.move_to_end(key)
                return t
            t = DrawTable(self, cdf_builder())
            self._tables[key] = t
            while len(self._tables) > 64:
                _, old = self._tables.popitem(last=False)
                old.close()
            return t

    # -- kernels -------------------------------------------------------------
    def run_replicates(self, table: DrawTable, support_k: int | None, gamma: float, n: int, base_seed: int,
                       repetition: int, first: int, count: int, ks, gamma_hat, status) -> None:
        """Enqueue replicates [first, first+count) into device tensors (float64, float64, uint8)."""
        cell = _native.ZksCell(
            support_k=0 if support_k is None else int(support_k),
            reserved=0,
            gamma=float(gamma),
            n=int(n),
            base_seed=int(base_seed),
            repetition=int(repetition),
            first=int(first),
            count=int(count),
        )
        self.bind_stream()
        _native.check(
            self.lib.zks_run_replicates(
                self.handle, table.handle, ctypes.byref(cell), ks.data_ptr(), gamma_hat.data_ptr(), status.data_ptr()
            )
        )

    def run_cells(self, tables, support_k: int | None, gammas, n: int, base_seed: int, repetition: int, first: int,
                  count: int, outs) -> None:
        """Enqueue replicates [first, first+count) of the cells of one sweep row (same n, support,
        seed, repetition; gammas differ; <= 32 cells): ``outs[j]`` = (ks, gamma_hat, status) device
        tensors of cell j.  Each replicate stream is drawn once for all cells (zks_run_cells)."""
        m = len(gammas)
        cells = (_native.ZksCell * m)(*[
            _native.ZksCell(support_k=0 if support_k is None else int(support_k), reserved=0, gamma=float(g), n=int(n),
                            base_seed=int(base_seed), repetition=int(repetition), first=int(first), count=int(count))
            for g in gammas])
        vp = ctypes.c_void_p
        handles = (vp * m)(*[t.handle.value for t in tables])
        ks = (vp * m)(*[o[0].data_ptr() for o in outs])
        gh = (vp * m)(*[o[1].data_ptr() for o in outs])
        st = (vp * m)(*[o[2].data_ptr() for o in outs])
        self.bind_stream()
        _native.check(self.lib.zks_run_cells(self.handle, m, handles, cells, ks, gh, st))

    def select_ranks(self, values, ranks: list[int], out=None):
        """Order statistics of a device float64 tensor at zero-based ranks.

        With ``out`` (device float64 tensor) the call is asynchronous; otherwise it returns a
        list of floats.
        """
        r = np.ascontiguousarray(ranks, dtype=np.int64)
        self.bind_stream()
        if out is not None:
            _native.check(
                self.lib.zks_select_ranks_async(self.handle, values.data_ptr(), values.numel(), r.ctypes.data, r.size,
                                                out.data_ptr())
            )
            return out
        res = np.empty(r.size, dtype=np.float64)
        _native.check(
            self.lib.zks_select_ranks(self.handle, values.data_ptr(), values.numel(), r.ctypes.data, r.size,
                                      res.ctypes.data)
        )
        return [float(x) for x in res]

    def select_many(self, jobs) -> None:
        """Asynchronous batched selection: ``jobs`` = [(values, ranks, out[, status, worst])] with
        device float64 ``values`` / ``out`` tensors and the same number (<= 16) of ranks each;
        with a device uint8 ``status`` tensor (as long as ``values``), its maximum lands in the
        one-element ``worst`` tensor.  One launch per 24 arrays."""
        jobs = list(jobs)
        for j0 in range(0, len(jobs), 24):
            part = jobs[j0 : j0 + 24]
            nr = len(part[0][1])
            ptrs = (ctypes.c_void_p * len(part))(*[j[0].data_ptr() for j in part])
            outs = (ctypes.c_void_p * len(part))(*[j[2].data_ptr() for j in part])
            sts = (ctypes.c_void_p * len(part))(*[j[3].data_ptr() if len(j) > 3 else None for j in part])
            worst = (ctypes.c_void_p * len(part))(*[j[4].data_ptr() if len(j) > 3 else None for j in part])
            counts = np.ascontiguousarray([j[0].numel() for j in part], dtype=np.int64)
            ranks = np.ascontiguousarray([list(j[1]) for j in part], dtype=np.int64)
            if ranks.shape[1] != nr:
                raise ValueError("select_many: every job needs the same number of ranks")
            for j in part:
                if len(j) > 3 and j[3].numel() != j[0].numel():
                    raise ValueError("select_many: status and values differ in length")
            self.bind_stream()
            _native.check(self.lib.zks_select_ranks_batch(self.handle, ptrs, counts.ctypes.data, len(part),
                                                          ranks.ctypes.data, nr, outs, sts, worst))

    def select_dist(self, jobs, total: int, reduce) -> None:
        """Batched selection over arrays sharded across processes: ``jobs`` as in select_many
        with this process's shard of each array (``total`` values in all, which the ranks refer
        to); ``reduce(t)`` must sum the device int32 tensor ``t`` over the processes in place
        (e.g. torch.distributed.all_reduce).  Per pass: local digit counts, reduce, pick."""
        torch = _torch()
        jobs = list(jobs)
        for j0 in range(0, len(jobs), 24):
            part = jobs[j0 : j0 + 24]
            nr = len(part[0][1])
            ptrs = (ctypes.c_void_p * len(part))(*[j[0].data_ptr() if j[0].numel() else None for j in part])
            outs = (ctypes.c_void_p * len(part))(*[j[2].data_ptr() for j in part])
            sts = (ctypes.c_void_p * len(part))(*[j[3].data_ptr() if len(j) > 3 and j[3].numel() else None
                                                  for j in part])
            worst = (ctypes.c_void_p * len(part))(*[j[4].data_ptr() if len(j) > 3 else None for j in part])
            counts = np.ascontiguousarray([j[0].numel() for j in part], dtype=np.int64)
            totals = np.full(len(part), int(total), dtype=np.int64)
            ranks = np.ascontiguousarray([list(j[1]) for j in part], dtype=np.int64)
            if ranks.shape[1] != nr:
                raise ValueError("select_dist: every job needs the same number of ranks")
            self.bind_stream()
            _native.check(self.lib.zks_select_dist_begin(self.handle, ptrs, counts.ctypes.data, totals.ctypes.data,
                                                         len(part), ranks.ctypes.data, nr, outs, sts, worst))
            hist = torch.empty(len(part) * nr * 256, dtype=torch.int32, device=part[0][2].device)
            for p in range(8):
                hist.zero_()
                _native.check(self.lib.zks_select_dist_count(self.handle, p, hist.data_ptr()))
                reduce(hist)
                self.bind_stream()
                _native.check(self.lib.zks_select_dist_pick(self.handle, p, hist.data_ptr()))
            _native.check(self.lib.zks_select_dist_end(self.handle))

    def normaliser(self, gamma: float, support_k: int | None) -> float:
        out = ctypes.c_double()
        self.bind_stream()
        _native.check(self.lib.zks_normaliser(self.handle, float(gamma), 0 if support_k is None else int(support_k),
                                              ctypes.byref(out)))
        return out.value

    def uniforms(self, seed: int, repetition: int, index: int, count: int, out) -> None:
        self.bind_stream()
        _native.check(self.lib.zks_stream_uniforms(self.handle, int(seed), int(repetition), int(index), int(count),
                                                   out.data_ptr()))

    def set_rng(self, kind: str) -> None:
        """Replicate streams: "numpy" (bit-exact with the reference, default) or "philox4x32"
        (opt-in fast generator, Monte Carlo parity only)."""
        kinds = {"numpy": 0, "philox4x32": 1}
        if kind not in kinds:
            raise ValueError(f"unknown stream kind {kind!r}; expected one of {sorted(kinds)}")
        _native.check(self.lib.zks_engine_set_rng(self.handle, kinds[kind]))
        self.rng = kind

    def set_chunk_bytes(self, nbytes: int = 0) -> None:
        """Budget of one chunk of pre-drawn rows (0 = 40 % of the free device memory, at most 48 GiB);
        results never depend on it."""
        _native.check(self.lib.zks_engine_set_chunk_bytes(self.handle, int(nbytes)))

    def uniforms_key(self, k0: int, k1: int, count: int, out) -> None:
        """Uniforms of an explicit Philox key (a host-derived SeedSequence of any other key)."""
        self.bind_stream()
        _native.check(self.lib.zks_stream_uniforms_key(self.handle, int(k0), int(k1), int(count), out.data_ptr()))

    def draw(self, table: DrawTable, u, out) -> None:
        self.bind_stream()
        _native.check(self.lib.zks_draw(self.handle, table.handle, u.data_ptr(), u.numel(), out.data_ptr()))

    # -- user samples / series ------------------------------------------------
    @staticmethod
    def _settings(settings):
        if settings is None:
            return None
        lo, hi = settings.bracket
        return _native.ZksMleSettings(float(settings.initial_guess), float(settings.absolute_tolerance),
                                      int(settings.max_iterations), 0, float(lo), float(hi))

    def fit_samples(self, support_k, values, offsets, mode, settings=None, gamma_in=None, norm_in=None) -> dict:
        """zks_fit_samples over device int64 ``values`` split by device int64 ``offsets``."""
        torch = _torch()
        ns = offsets.numel() - 1
        dev = values.device
        out = {
            "log_mean": torch.empty(ns, dtype=torch.float64, device=dev),
            "gamma": torch.empty(ns, dtype=torch.float64, device=dev),
            "ks": torch.empty(ns, dtype=torch.float64, device=dev),
            "argmax": torch.empty(ns, dtype=torch.int64, device=dev),
            "status": torch.empty(ns, dtype=torch.uint8, device=dev),
        }
        st = self._settings(settings)
        self.bind_stream()
        _native.check(self.lib.zks_fit_samples(
            self.handle, 0 if support_k is None else int(support_k), values.data_ptr(), offsets.data_ptr(), ns,
            int(mode), ctypes.byref(st) if st is not None else None,
            gamma_in.data_ptr() if gamma_in is not None else None, norm_in.data_ptr() if norm_in is not None else None,
            out["log_mean"].data_ptr(), out["gamma"].data_ptr(), out["ks"].data_ptr(), out["argmax"].data_ptr(),
            out["status"].data_ptr()))
        return out

    def series(self, support_k, gammas):
        """(s0, s1, s2, normaliser) rows at device float64 ``gammas`` (reference formulas)."""
        torch = _torch()
        out = torch.empty((gammas.numel(), 4), dtype=torch.float64, device=gammas.device)
        self.bind_stream()
        _native.check(self.lib.zks_series_eval(self.handle, 0 if support_k is None else int(support_k),
                                               gammas.data_ptr(), gammas.numel(), out.data_ptr()))
        return out

    def tail_mass(self, gamma: float, starts):
        """sum_{k >= s} k^-gamma at device float64 ``starts`` (each > 64)."""
        torch = _torch()
        out = torch.empty_like(starts)
        self.bind_stream()
        _native.check(self.lib.zks_tail_mass(self.handle, float(gamma), starts.data_ptr(), starts.numel(),
                                             out.data_ptr()))
        return out

    def solve(self, support_k, targets, settings=None, bisect_only=False):
        torch = _torch()
        g = torch.empty_like(targets)
        st = torch.empty(targets.numel(), dtype=torch.uint8, device=targets.device)
        s = self._settings(settings)
        self.bind_stream()
        _native.check(self.lib.zks_solve_exponents(self.handle, 0 if support_k is None else int(support_k),
                                                   targets.data_ptr(), targets.numel(),
                                                   ctypes.byref(s) if s is not None else None, int(bisect_only),
                                                   g.data_ptr(), st.data_ptr()))
        return g, st

    # -- diagnostics ---------------------------------------------------------
    def set_counters(self, counters) -> None:
        """Count replicate-kernel work into a device uint64/int64 tensor of 8 (None = off)."""
        ptr = None if counters is None else ctypes.c_void_p(counters.data_ptr())
        _native.check(self.lib.zks_engine_set_counters(self.handle, ptr))

    def set_mle_mode(self, direct: bool) -> None:
        """Model moments by direct summation (validation) instead of the fit tables."""
        _native.check(self.lib.zks_engine_set_mle_mode(self.handle, _native.MLE_DIRECT if direct else _native.MLE_TABLE))

    def fit_eval(self, support_k: int | None, x):
        """Fit-table values (mu, m2, norm) at device float64 points ``x``."""
        torch = _torch()
        mu, m2, nrm = (torch.empty_like(x) for _ in range(3))
        self.bind_stream()
        _native.check(self.lib.zks_fit_eval(self.handle, 0 if support_k is None else int(support_k), x.data_ptr(),
                                            x.numel(), mu.data_ptr(), m2.data_ptr(), nrm.data_ptr()))
        return mu, m2, nrm

    def probe_peaks(self) -> dict:
        """Measured pipe peaks of this device: DFMA FLOP/s, FP64 exp/s, 64-bit mulhilo/s."""
        out = (ctypes.c_double * 3)()
        self.bind_stream()
        _native.check(self.lib.zks_probe_peaks(self.handle, out))
        return {"dfma_flops": out[0], "exp_per_s": out[1], "mul64_per_s": out[2]}

    def clear_tables(self) -> None:
        with self._lock:
            for t in self._tables.values():
                t.close()
            self._tables.clear()

    def close(self) -> None:
        for t in self._tables.values():
            t.close()
        self._tables.clear()
        if self.handle:
            self.lib.zks_engine_destroy(self.handle)
            self.handle = None


_ENGINES: dict[int, Engine] = {}
_ENGINES_LOCK = threading.Lock()


def get_engine(device: int | None = None) -> Engine:
    """Process-wide engine of ``device`` (default: torch's current device)."""
    torch = _torch()
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("zipfks_b200 needs a CUDA device (sm_100a); none is visible")
        device = torch.cuda.current_device()
    with _ENGINES_LOCK:
        eng = _ENGINES.get(device)
        if eng is None:
            eng = Engine(device)
            _ENGINES[device] = eng
        return eng
