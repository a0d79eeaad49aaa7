"""paper_2604_15768_b200 -- B200-native selected-CI hot path (QiankunNet-cuSCI,
arXiv 2604.15768): gen_coupled -> dedup_global -> merge_space.

Thin Python binding over the C ABI of libcusci.so (include/cusci.h): argument
marshalling only, every step runs in the library's sm_100a kernels.  PyTorch
supplies device memory (through the allocator callback), streams and process
groups.  There is no CPU fallback: importing this package on a machine without
the built library raises, and every call needs a CUDA device.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from ._lib import CUSCI_ERRORS, CusciError, lib, LIB_PATH  # noqa: F401

__all__ = ["Space", "DeviceIntegrals", "Context", "Pool", "Records", "HostRecords", "CusciError", "LIB_PATH",
           "gen_coupled_bound"]


class _Space(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int32), ("n_alpha", ctypes.c_int32), ("n_beta", ctypes.c_int32),
                ("words", ctypes.c_int32)]


class _Integrals(ctypes.Structure):
    _fields_ = [("n_spatial", ctypes.c_int32), ("h", ctypes.c_void_p), ("eri", ctypes.c_void_p)]


class _Records(ctypes.Structure):
    _fields_ = [("keys", ctypes.c_void_p), ("hij", ctypes.c_void_p), ("src", ctypes.c_void_p),
                ("phase", ctypes.c_void_p), ("capacity", ctypes.c_uint64), ("count", ctypes.c_uint64)]


class _Keys(ctypes.Structure):
    _fields_ = [("keys", ctypes.c_void_p), ("count", ctypes.c_uint64)]


class _StreamCfg(ctypes.Structure):
    _fields_ = [("batch_parents", ctypes.c_uint64), ("batch_records", ctypes.c_uint64), ("host_keys", ctypes.c_void_p),
                ("host_hij", ctypes.c_void_p), ("host_src", ctypes.c_void_p), ("host_capacity", ctypes.c_uint64)]


class _GrowStats(ctypes.Structure):
    _fields_ = [("records", ctypes.c_uint64), ("unique", ctypes.c_uint64), ("candidates", ctypes.c_uint64),
                ("selected", ctypes.c_uint64), ("space_before", ctypes.c_uint64), ("space_after", ctypes.c_uint64),
                ("ms", ctypes.c_double)]


class _StreamStats(ctypes.Structure):
    _fields_ = [("batches", ctypes.c_uint64), ("records", ctypes.c_uint64), ("unique", ctypes.c_uint64),
                ("ms_wall", ctypes.c_double), ("ms_h2d", ctypes.c_double), ("ms_compute", ctypes.c_double),
                ("ms_d2h", ctypes.c_double), ("h2d_bytes", ctypes.c_uint64), ("d2h_bytes", ctypes.c_uint64),
                ("peak_device_bytes", ctypes.c_uint64)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


class Space:
    """m spin orbitals (interleaved alpha/beta), n_alpha / n_beta electrons."""

    def __init__(self, m: int, n_alpha: int, n_beta: int):
        self.m, self.n_alpha, self.n_beta = int(m), int(n_alpha), int(n_beta)
        self.words = 1 if self.m <= 64 else 2

    def _c(self) -> _Space:
        return _Space(self.m, self.n_alpha, self.n_beta, self.words)

    def __repr__(self):
        return f"Space(m={self.m}, n_alpha={self.n_alpha}, n_beta={self.n_beta}, words={self.words})"


class DeviceIntegrals:
    """h [K,K] and packed (PQ|RS) as float64 CUDA tensors (kept alive here)."""

    def __init__(self, h, eri, device="cuda"):
        self.h = torch.as_tensor(h, dtype=torch.float64).to(device).contiguous()
        self.eri = torch.as_tensor(eri, dtype=torch.float64).to(device).contiguous()
        self.n_spatial = int(self.h.shape[0])

    def _c(self) -> _Integrals:
        return _Integrals(self.n_spatial, self.h.data_ptr(), self.eri.data_ptr())


def gen_coupled_bound(space: Space, n_parents: int) -> int:
    sp = space._c()
    return int(lib().gen_coupled_bound(ctypes.byref(sp), int(n_parents)))


class Records:
    """Output of gen_coupled: keys uint64 [count, W], hij float64 [count],
    src uint32-as-int32 [count] (or None), phase int8 [count] (or None)."""

    def __init__(self, keys, hij, src, phase, count):
        self.keys, self.hij, self.src, self.phase, self.count = keys, hij, src, phase, count


class HostRecords:
    """The host-resident "original set" of the streaming stages:
    pinned keys uint64 [capacity, W], hij float64 [capacity], src int32 (global
    parent index) [capacity]; `count` = records held."""

    def __init__(self, capacity: int, W: int):
        self.capacity, self.W, self.count = int(capacity), int(W), 0
        self.keys = torch.empty((self.capacity, W), dtype=torch.uint64, pin_memory=True)
        self.hij = torch.empty(self.capacity, dtype=torch.float64, pin_memory=True)
        self.src = torch.empty(self.capacity, dtype=torch.int32, pin_memory=True)

    def _cfg(self, batch_parents: int = 0, batch_records: int = 0) -> "_StreamCfg":
        return _StreamCfg(int(batch_parents), int(batch_records), self.keys.data_ptr(), self.hij.data_ptr(),
                          self.src.data_ptr(), self.capacity)


def _host_u64(t: torch.Tensor, W: int) -> torch.Tensor:
    if t.dtype != torch.uint64 or t.is_cuda:
        raise TypeError("host parents must be a CPU torch.uint64 tensor (pinned for overlap)")
    return t.reshape(-1, W).contiguous()


_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
_FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)


def _as_u64_2d(t: torch.Tensor, W: int) -> torch.Tensor:
    if t.dtype != torch.uint64:
        raise TypeError("configuration keys must be torch.uint64")
    if not t.is_cuda:
        raise ValueError("configuration keys must be a CUDA tensor")
    return t.reshape(-1, W).contiguous()


class Context:
    """One library context per (process, GPU): stream, NCCL communicator,
    output allocator (torch caching allocator), cached Hamiltonian prep."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 stream: torch.cuda.Stream | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2604_15768_b200 needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._live: dict[int, torch.Tensor] = {}

        def _alloc(nbytes, _stream, _user):
            try:
                with torch.cuda.stream(self.stream):
                    t = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
            except RuntimeError:
                return None
            p = t.data_ptr()
            self._live[p] = t
            return p

        def _free(ptr, _user):
            self._live.pop(ptr, None)

        self._alloc_cb = _ALLOC_FN(_alloc)
        self._free_cb = _FREE_FN(_free)
        idbuf = None
        if world > 1 and nccl_id is None:
            raise ValueError("world > 1 needs the 128-byte NCCL unique id")
        if nccl_id is not None:   # world = 1 with an id: a 1-rank communicator (force_collective)
            if len(nccl_id) != 128:
                raise ValueError("the NCCL unique id is 128 bytes")
            idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        ctx = ctypes.c_void_p()
        rc = lib().cusci_init(ctypes.byref(ctx), device, rank, world, idbuf, ctypes.c_void_p(self.stream.cuda_stream),
                              self._alloc_cb, self._free_cb, None)
        if rc != 0:
            raise CusciError(rc, "cusci_init failed")
        self._ctx = ctx
        self.rank, self.world = rank, world
        self._ints = None   # the integrals of the library's cached Hamiltonian prep (kept alive)

    # ------------------------------------------------------------------ plumbing
    def close(self):
        if getattr(self, "_ctx", None):
            lib().cusci_finalize(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int, what: str):
        if rc != 0:
            msg = lib().cusci_last_error(self._ctx).decode(errors="replace")
            raise CusciError(rc, f"{what}: {msg}")

    def _take(self, ptr: int | None, count: int, W: int) -> torch.Tensor:
        if not ptr:
            return torch.empty((0, W), dtype=torch.uint64, device=self.device)
        t = self._live.pop(ptr)
        return t.view(torch.uint64)[: count * W].view(count, W)

    @property
    def kernel_launches(self) -> int:
        return int(lib().cusci_kernel_launches(self._ctx))

    def profile(self, on: bool = True):
        """Enable/disable the library's per-kernel-class CUDA-event profiler."""
        lib().cusci_profile_enable(self._ctx, 1 if on else 0)

    def profile_read(self) -> dict:
        """{kernel class: (milliseconds, launches)} since the last read."""
        from ._lib import PROFILE_TAGS
        n = len(PROFILE_TAGS)
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_uint64 * n)()
        self._check(lib().cusci_profile_read(self._ctx, ms, cnt, n), "cusci_profile_read")
        return {t: (ms[i], int(cnt[i])) for i, t in enumerate(PROFILE_TAGS) if cnt[i]}

    def dedup_stats(self, reset: bool = True) -> dict:
        """Local-dedup plan statistics since the last reset (cusci_dedup_stats)."""
        st = (ctypes.c_uint64 * 8)()
        self._check(lib().cusci_dedup_stats(self._ctx, st, 1 if reset else 0), "cusci_dedup_stats")
        return dict(zip(("calls", "keys_in", "key_passes", "keys_out", "buckets", "slow_path_calls", "hist_keys",
                         "hist_free_keys"), (int(x) for x in st)))

    def release_cached(self):
        """Return the library's cached device memory (scratch arena, freed pool blocks)."""
        self._check(lib().cusci_release_cached(self._ctx), "cusci_release_cached")

    def invalidate_integrals(self):
        lib().cusci_invalidate_integrals(self._ctx)
        self._ints = None

    def _use_integrals(self, ints: "DeviceIntegrals"):
        # the library caches its prep by pointer: keep these integrals alive while
        # cached, and drop the cache when another integrals object comes in
        if ints is not self._ints:
            lib().cusci_invalidate_integrals(self._ctx)
            self._ints = ints

    def force_collective(self, on: bool = True):
        """Run the collective protocol (status-carrying count exchange, NCCL
        payload exchange) even at world = 1 (needs Context(..., nccl_id=...))."""
        from ._lib import CUSCI_OPT_FORCE_COLLECTIVE
        self._check(lib().cusci_set_option(self._ctx, CUSCI_OPT_FORCE_COLLECTIVE, 1 if on else 0), "cusci_set_option")

    def contract_partition(self, mode: int = 0):
        """energy_contract's pi-partition of the records: 1 on, 0 (default) / -1 off."""
        from ._lib import CUSCI_OPT_CONTRACT_PARTITION
        self._check(lib().cusci_set_option(self._ctx, CUSCI_OPT_CONTRACT_PARTITION, int(mode)), "cusci_set_option")

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        rc = lib().cusci_nccl_unique_id(buf)
        if rc != 0:
            raise CusciError(rc, "ncclGetUniqueId failed")
        return buf.raw

    # ------------------------------------------------------------------ step 1
    def gen_coupled(self, space: Space, parents: torch.Tensor, ints: DeviceIntegrals, threshold: float = 0.0,
                    capacity: int | None = None, with_src: bool = True, with_phase: bool = False,
                    out: Records | None = None) -> Records:
        """Coupled configurations of every parent with H_ij (include/cusci.h gen_coupled).
        `out` (optional) supplies preallocated buffers (keys [cap, W], hij [cap], src, phase)."""
        W = space.words
        par = _as_u64_2d(parents, W)
        n = par.shape[0]
        if out is None:
            if capacity is None:
                capacity = self.gen_coupled_count(space, par, ints, threshold)
            cap = int(capacity)
            keys = torch.empty((cap, W), dtype=torch.uint64, device=self.device)
            hij = torch.empty(cap, dtype=torch.float64, device=self.device)
            src = torch.empty(cap, dtype=torch.int32, device=self.device) if with_src else None
            phase = torch.empty(cap, dtype=torch.int8, device=self.device) if with_phase else None
        else:
            keys, hij, src, phase = out.keys, out.hij, out.src, out.phase
            cap = int(keys.shape[0])
        self._use_integrals(ints)
        rec = _Records(keys.data_ptr(), hij.data_ptr(), src.data_ptr() if src is not None else None,
                       phase.data_ptr() if phase is not None else None, cap, 0)
        sp, ci = space._c(), ints._c()
        rc = lib().gen_coupled(self._ctx, ctypes.byref(sp), ctypes.c_void_p(par.data_ptr()), n, ctypes.byref(ci),
                               float(threshold), ctypes.byref(rec))
        self._check(rc, "gen_coupled")
        c = int(rec.count)
        return Records(keys[:c], hij[:c], src[:c] if src is not None else None,
                       phase[:c] if phase is not None else None, c)

    def gen_coupled_count(self, space: Space, parents: torch.Tensor, ints: DeviceIntegrals,
                          threshold: float = 0.0) -> int:
        par = _as_u64_2d(parents, space.words)
        self._use_integrals(ints)
        cnt = ctypes.c_uint64(0)
        sp, ci = space._c(), ints._c()
        rc = lib().gen_coupled_count(self._ctx, ctypes.byref(sp), ctypes.c_void_p(par.data_ptr()), par.shape[0],
                                     ctypes.byref(ci), float(threshold), ctypes.byref(cnt))
        self._check(rc, "gen_coupled_count")
        return int(cnt.value)

    # ------------------------------------------------------------------ step 2
    def dedup_global(self, space: Space, configs: torch.Tensor) -> torch.Tensor:
        """Sorted unique keys owned by this rank (collective when world > 1)."""
        W = space.words
        cfg = _as_u64_2d(configs, W)
        k = _Keys()
        sp = space._c()
        rc = lib().dedup_global(self._ctx, ctypes.byref(sp), ctypes.c_void_p(cfg.data_ptr()), cfg.shape[0],
                                ctypes.byref(k))
        self._check(rc, "dedup_global")
        return self._take(k.keys, int(k.count), W)

    def dedup_partition(self, space: Space, configs: torch.Tensor, n_owners: int):
        """(bins [sum counts, W] back to back by owner, counts list)."""
        W = space.words
        cfg = _as_u64_2d(configs, W)
        k = _Keys()
        counts = (ctypes.c_uint64 * n_owners)()
        sp = space._c()
        rc = lib().dedup_partition(self._ctx, ctypes.byref(sp), ctypes.c_void_p(cfg.data_ptr()), cfg.shape[0],
                                   n_owners, ctypes.byref(k), counts)
        self._check(rc, "dedup_partition")
        return self._take(k.keys, int(k.count), W), [int(c) for c in counts]

    # ---- the paper's regular-sampling sorted dedup (PAPER.md :448-462)
    def dedup_sorted(self, space: Space, configs: torch.Tensor, n_samples: int = 1024, want_splitters: bool = False):
        """COLLECTIVE: this rank's shard of the distinct keys in the big-integer key order
        (regular-sampling splitters); with want_splitters also the (P-1, W) host splitters."""
        W = space.words
        cfg = _as_u64_2d(configs, W)
        k = _Keys()
        sp = space._c()
        nsp = max(self.world - 1, 1) * W
        spl = (ctypes.c_uint64 * nsp)()
        rc = lib().dedup_sorted(self._ctx, ctypes.byref(sp), ctypes.c_void_p(cfg.data_ptr()), cfg.shape[0], n_samples,
                                ctypes.byref(k), spl)
        self._check(rc, "dedup_sorted")
        out = self._take(k.keys, int(k.count), W)
        if want_splitters:
            return out, np.array(spl[:(self.world - 1) * W], dtype=np.uint64).reshape(-1, W)
        return out

    def sort_unique(self, space: Space, configs: torch.Tensor) -> torch.Tensor:
        """Sorted (big-integer order) unique keys of configs (Step 1 of the paper's dedup)."""
        W = space.words
        cfg = _as_u64_2d(configs, W)
        k = _Keys()
        sp = space._c()
        self._check(lib().sort_unique(self._ctx, ctypes.byref(sp), ctypes.c_void_p(cfg.data_ptr()), cfg.shape[0],
                                      ctypes.byref(k)), "sort_unique")
        return self._take(k.keys, int(k.count), W)

    def regular_samples(self, space: Space, sorted_keys: torch.Tensor, n_samples: int) -> torch.Tensor:
        W = space.words
        srt = _as_u64_2d(sorted_keys, W)
        out = torch.empty((max(min(n_samples, srt.shape[0]), 1), W), dtype=torch.uint64, device=self.device)
        taken = ctypes.c_uint64(0)
        sp = space._c()
        self._check(lib().regular_samples(self._ctx, ctypes.byref(sp), ctypes.c_void_p(srt.data_ptr()), srt.shape[0],
                                          n_samples, ctypes.c_void_p(out.data_ptr()), ctypes.byref(taken)),
                    "regular_samples")
        return out[:taken.value]

    def select_splitters(self, space: Space, samples: torch.Tensor, n_parts: int) -> torch.Tensor:
        W = space.words
        smp = _as_u64_2d(samples, W)
        out = torch.zeros((max(n_parts - 1, 1), W), dtype=torch.uint64, device=self.device)
        sp = space._c()
        self._check(lib().select_splitters(self._ctx, ctypes.byref(sp), ctypes.c_void_p(smp.data_ptr()), smp.shape[0],
                                           n_parts, ctypes.c_void_p(out.data_ptr())), "select_splitters")
        return out[:n_parts - 1]

    def split_bounds(self, space: Space, sorted_keys: torch.Tensor, splitters: torch.Tensor, n_parts: int):
        W = space.words
        srt = _as_u64_2d(sorted_keys, W)
        spl = _as_u64_2d(splitters, W) if n_parts > 1 else srt
        b = (ctypes.c_uint64 * (n_parts + 1))()
        sp = space._c()
        self._check(lib().split_bounds(self._ctx, ctypes.byref(sp), ctypes.c_void_p(srt.data_ptr()), srt.shape[0],
                                       ctypes.c_void_p(spl.data_ptr()), n_parts, b), "split_bounds")
        return [int(x) for x in b]

    def dedup_finalize(self, space: Space, keys: torch.Tensor) -> torch.Tensor:
        W = space.words
        cfg = _as_u64_2d(keys, W)
        k = _Keys()
        sp = space._c()
        rc = lib().dedup_finalize(self._ctx, ctypes.byref(sp), ctypes.c_void_p(cfg.data_ptr()), cfg.shape[0],
                                  ctypes.byref(k))
        self._check(rc, "dedup_finalize")
        return self._take(k.keys, int(k.count), W)

    def dedup_finalize_runs(self, space: Space, keys: torch.Tensor, run_counts) -> torch.Tensor:
        """Owner-side unique of runs received back to back, each strictly
        increasing in the hash order (dedup_partition bins)."""
        W = space.words
        cfg = _as_u64_2d(keys, W)
        counts = (ctypes.c_uint64 * len(run_counts))(*[int(c) for c in run_counts])
        if sum(int(c) for c in run_counts) != cfg.shape[0]:
            raise ValueError("run_counts must sum to the number of keys")
        k = _Keys()
        sp = space._c()
        rc = lib().dedup_finalize_runs(self._ctx, ctypes.byref(sp), ctypes.c_void_p(cfg.data_ptr()), counts,
                                       len(run_counts), ctypes.byref(k))
        self._check(rc, "dedup_finalize_runs")
        return self._take(k.keys, int(k.count), W)

    # ---- SCI growth with the heat-bath surrogate (Sec 2.2)
    def sci_grow_step(self, space: Space, pool: "Pool", psi: torch.Tensor, ints: DeviceIntegrals,
                      threshold: float, K: int):
        """One iteration S <- S u top-K(C \\ S by heat-bath score); returns (psi over the
        new S in pool order, stats)."""
        psi = psi.contiguous()
        if psi.dtype != torch.float64 or not psi.is_cuda or psi.numel() != len(pool):
            raise ValueError("psi must be a CUDA float64 tensor aligned with the pool")
        self._use_integrals(ints)
        cap = len(pool) + int(K)
        out = torch.empty(max(cap, 1), dtype=torch.float64, device=self.device)
        st = _GrowStats()
        sp, ci = space._c(), ints._c()
        rc = lib().sci_grow_step(self._ctx, ctypes.byref(sp), pool._pool, ctypes.c_void_p(psi.data_ptr()),
                                 ctypes.byref(ci), float(threshold), int(K), ctypes.c_void_p(out.data_ptr()), cap,
                                 ctypes.byref(st))
        self._check(rc, "sci_grow_step")
        return out[: st.space_after], {f: getattr(st, f) for f, _ in st._fields_}

    # ---- memory-centric streaming (Sec 4.3)
    def stream_generate(self, space: Space, parents_host: torch.Tensor, ints: DeviceIntegrals, threshold: float,
                        batch_parents: int, unique_pool: "Pool", host: "HostRecords | None" = None,
                        batch_records: int = 0) -> dict:
        """Stage 1: parent mini-batches -> gen_coupled -> dedup_global -> merge_space(unique_pool),
        with H2D prefetch and (if `host`) D2H offload of the records on their own streams.
        batch_records: record-slot capacity hint (0: count every batch first)."""
        par = _host_u64(parents_host, space.words)
        self._use_integrals(ints)
        cfg = host._cfg(batch_parents, batch_records) if host is not None else \
            _StreamCfg(int(batch_parents), int(batch_records), None, None, None, 0)
        st = _StreamStats()
        sp, ci = space._c(), ints._c()
        rc = lib().stream_generate(self._ctx, ctypes.byref(sp), ctypes.c_void_p(par.data_ptr()), par.shape[0],
                                   ctypes.byref(ci), float(threshold), ctypes.byref(cfg), unique_pool._pool,
                                   ctypes.byref(st))
        if host is not None:
            host.count = min(int(st.records), host.capacity)
        self._check(rc, "stream_generate")
        return st.as_dict()

    def stream_energy(self, space: Space, host: "HostRecords", n_parents: int, space_keys: torch.Tensor,
                      psi: torch.Tensor, batch_records: int, e: torch.Tensor | None = None):
        """Stage 3 (reload): the host original set streamed back in record batches and
        contracted; returns (e, n_missing, stats)."""
        sk = _as_u64_2d(space_keys, space.words)
        psi = psi.contiguous()
        if e is None:
            e = torch.empty(max(int(n_parents), 0), dtype=torch.float64, device=self.device)
        miss = ctypes.c_uint64()
        st = _StreamStats()
        cfg = host._cfg(0, batch_records)
        rc = lib().stream_energy(self._ctx, ctypes.byref(space._c()), ctypes.byref(cfg), host.count, int(n_parents),
                                 ctypes.c_void_p(sk.data_ptr()), sk.shape[0], ctypes.c_void_p(psi.data_ptr()),
                                 ctypes.c_void_p(e.data_ptr()), ctypes.byref(miss), ctypes.byref(st))
        self._check(rc, "stream_energy")
        return e, int(miss.value), st.as_dict()

    def stream_energy_regen(self, space: Space, parents_host: torch.Tensor, ints: DeviceIntegrals, threshold: float,
                            batch_parents: int, space_keys: torch.Tensor, psi: torch.Tensor,
                            e: torch.Tensor | None = None):
        """Stage 3 (regenerate): the records of each parent batch generated again on the
        device and contracted; returns (e, n_missing, stats)."""
        par = _host_u64(parents_host, space.words)
        self._use_integrals(ints)
        sk = _as_u64_2d(space_keys, space.words)
        psi = psi.contiguous()
        if e is None:
            e = torch.empty(max(par.shape[0], 0), dtype=torch.float64, device=self.device)
        miss = ctypes.c_uint64()
        st = _StreamStats()
        cfg = _StreamCfg(int(batch_parents), 0, None, None, None, 0)
        sp, ci = space._c(), ints._c()
        rc = lib().stream_energy_regen(self._ctx, ctypes.byref(sp), ctypes.c_void_p(par.data_ptr()), par.shape[0],
                                       ctypes.byref(ci), float(threshold), ctypes.byref(cfg),
                                       ctypes.c_void_p(sk.data_ptr()), sk.shape[0], ctypes.c_void_p(psi.data_ptr()),
                                       ctypes.c_void_p(e.data_ptr()), ctypes.byref(miss), ctypes.byref(st))
        self._check(rc, "stream_energy_regen")
        return e, int(miss.value), st.as_dict()

    # ------------------------------------------------------------------ step 3
    def pool(self, space: Space, capacity: int = 1 << 20) -> "Pool":
        return Pool(self, space, capacity)

    def merge_pool(self, dst: "Pool", src: "Pool", want_inserted: bool = False):
        """dst <- dst u src (cusci_pool_merge): src's keys are read in place and,
        being a pool's, are not re-validated."""
        k = _Keys()
        rc = lib().cusci_pool_merge(self._ctx, dst._pool, src._pool, ctypes.byref(k) if want_inserted else None)
        self._check(rc, "cusci_pool_merge")
        if want_inserted:
            return self._take(k.keys, int(k.count), dst.space.words)
        return None

    def merge_space(self, pool: "Pool", new_keys: torch.Tensor, want_inserted: bool = False):
        W = pool.space.words
        nk = _as_u64_2d(new_keys, W)
        k = _Keys()
        rc = lib().merge_space(self._ctx, pool._pool, ctypes.c_void_p(nk.data_ptr()), nk.shape[0],
                               ctypes.byref(k) if want_inserted else None)
        self._check(rc, "merge_space")
        if want_inserted:
            return self._take(k.keys, int(k.count), W)
        return None

    def energy_contract(self, space: Space, rec: "Records", n_parents: int, space_keys: torch.Tensor,
                        psi: torch.Tensor, e: torch.Tensor = None):
        """Stage-3 contraction (Eq. 5): e[s] = sum_{r: src_r = s} H_r psi[idx(key_r)]
        with the just-in-time reverse index into the hash-ordered unique set
        `space_keys` (psi aligned with it).  Returns (e float64 [n_parents], n_missing)."""
        W = space.words
        n = int(rec.count)
        keys = _as_u64_2d(rec.keys[:n], W)
        if rec.src is None:
            raise ValueError("energy_contract needs records with src")
        sk = _as_u64_2d(space_keys, W)
        psi = psi.contiguous()
        if psi.dtype != torch.float64 or psi.numel() != sk.shape[0]:
            raise ValueError("psi must be float64 and aligned with space_keys")
        if e is None:
            e = torch.empty(max(int(n_parents), 0), dtype=torch.float64, device=keys.device)
        elif e.dtype != torch.float64 or e.numel() < int(n_parents) or not e.is_contiguous() or not e.is_cuda:
            raise ValueError("e must be a contiguous CUDA float64 tensor with >= n_parents elements")
        miss = ctypes.c_uint64()
        rc = lib().energy_contract(self._ctx, ctypes.byref(space._c()), ctypes.c_void_p(keys.data_ptr()),
                                   ctypes.c_void_p(rec.hij.data_ptr()), ctypes.c_void_p(rec.src.data_ptr()), n,
                                   int(n_parents), ctypes.c_void_p(sk.data_ptr()), sk.shape[0],
                                   ctypes.c_void_p(psi.data_ptr()), ctypes.c_void_p(e.data_ptr()), ctypes.byref(miss))
        self._check(rc, "energy_contract")
        return e, int(miss.value)


class Pool:
    """GPU-resident sorted unique configuration shard (library owned)."""

    def __init__(self, ctx: Context, space: Space, capacity: int):
        self.ctx, self.space = ctx, space
        p = ctypes.c_void_p()
        sp = space._c()
        ctx._check(lib().cusci_pool_create(ctx._ctx, ctypes.byref(sp), int(capacity), ctypes.byref(p)),
                   "cusci_pool_create")
        self._pool = p

    def __len__(self) -> int:
        ptr, cnt = ctypes.c_void_p(), ctypes.c_uint64()
        lib().cusci_pool_view(self._pool, ctypes.byref(ptr), ctypes.byref(cnt))
        return int(cnt.value)

    def view(self):
        """(device pointer, count) of the pool's keys, valid until the next merge."""
        ptr, cnt = ctypes.c_void_p(), ctypes.c_uint64()
        lib().cusci_pool_view(self._pool, ctypes.byref(ptr), ctypes.byref(cnt))
        return ptr.value or 0, int(cnt.value)

    def clear(self):
        self.ctx._check(lib().cusci_pool_clear(self._pool), "cusci_pool_clear")

    def keys(self) -> torch.Tensor:
        """A copy of the pool's keys (uint64 [count, W])."""
        ptr, cnt = ctypes.c_void_p(), ctypes.c_uint64()
        lib().cusci_pool_view(self._pool, ctypes.byref(ptr), ctypes.byref(cnt))
        n, W = int(cnt.value), self.space.words
        out = torch.empty((n, W), dtype=torch.uint64, device=self.ctx.device)
        self.ctx._check(lib().cusci_pool_copy(self._pool, ctypes.c_void_p(out.data_ptr()), n), "cusci_pool_copy")
        return out

    def close(self):
        if getattr(self, "_pool", None):
            lib().cusci_pool_destroy(self._pool)
            self._pool = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
