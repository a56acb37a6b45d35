"""B200 system facade: one native context per GPU behind the reference's ``AgileSystem`` shape.

Reference: ``system.py:34-185`` builds devices, queue pairs, cache, service and API around a
discrete-event simulator and runs generator programs.  Here the same configuration tree builds a
native context (``agile_create``) that owns the HBM cache, the SQ/CQ rings, the completion
service and the emulated devices backed by host-pinned GPU-mapped page stores; workloads are
request arrays handed to fused kernels (``run_seq`` / ``run_reads`` / ``run_loop`` /
``run_gather`` / ``embbag``).  Counters keep the reference's names (``cache.hits``,
``service.stats.completions``, ``devices[d].bytes_read`` ...).
"""

from __future__ import annotations

import copy
import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .config import SystemConfig, config_text
from .trace import TraceRecorder, render_event_log

STAT_NAMES = ("hits", "misses", "fills", "writebacks", "resets", "attaches", "completions",
              "windows_rung", "drain_entries_rung", "bytes_read", "bytes_written", "fetched",
              "doorbells", "sq_full", "cqe_stalls", "barrier_count", "barrier_latency_sum",
              "retries", "enqueues", "lookups", "waits")

BLOCK = 4096
DEV_SHIFT = 36


def make_key(dev, blk):
    """Request key: dev << 36 | blk (numpy-vectorised)."""
    return (np.asarray(dev, dtype=np.uint64) << np.uint64(DEV_SHIFT)) | np.asarray(blk, dtype=np.uint64)


@dataclass
class ServiceStats:
    completions: int = 0
    windows_rung: int = 0
    drain_entries_rung: int = 0
    barrier_count: int = 0
    barrier_latency_sum: int = 0

    @property
    def mean_barrier_ns(self) -> float:
        return self.barrier_latency_sum / self.barrier_count if self.barrier_count else 0.0


class _CacheView:
    def __init__(self, s):
        self.hits, self.misses, self.fills = s["hits"], s["misses"], s["fills"]
        self.writebacks, self.resets, self.attaches = s["writebacks"], s["resets"], s["attaches"]


class _Store:
    def __init__(self, system, dev):
        self._system, self._dev = system, dev

    @property
    def num_blocks(self) -> int:
        return self._system._store_blocks(self._dev)

    @property
    def block_size(self) -> int:
        return BLOCK

    def view(self) -> np.ndarray:
        return self._system.store_view(self._dev)

    def read_block(self, blk: int) -> bytes:
        from .errors import OutOfRange
        if not 0 <= blk < self.num_blocks:
            raise OutOfRange(f"block {blk} out of range [0, {self.num_blocks})")
        return bytes(self.view()[blk])

    def write_block(self, blk: int, payload) -> None:
        from .errors import OutOfRange
        if not 0 <= blk < self.num_blocks:
            raise OutOfRange(f"block {blk} out of range [0, {self.num_blocks})")
        if len(payload) != BLOCK:
            raise ValueError("payload must be exactly one block")
        self.view()[blk] = np.frombuffer(bytes(payload), dtype=np.uint8)

    def load_image(self, path) -> None:
        self._system.load_image(self._dev, path)

    def save_image(self, path) -> None:
        self._system.save_image(self._dev, path)


class _Device:
    def __init__(self, system, dev):
        self.dev_idx = dev
        self.store = _Store(system, dev)
        self._system = system

    @property
    def bytes_read(self) -> int:
        return self._system.stats()["bytes_read"]   # aggregated over devices

    @property
    def bytes_written(self) -> int:
        return self._system.stats()["bytes_written"]


class AgileSystem:
    """Native B200 context for one GPU (drop-in shape of reference ``AgileSystem``)."""

    def __init__(self, cfg: SystemConfig | None = None, recorder: TraceRecorder | None = None,
                 device: int | None = None, trace_capacity: int = 1 << 22):
        self.cfg = copy.deepcopy(cfg) if cfg is not None else SystemConfig()
        if self.cfg.backend != "b200":
            raise ValueError("this package implements backend = b200 only")
        self.recorder = recorder
        self.block_size = self.cfg.device.block_size
        self._lib = _lib.load()
        if device is None:
            import torch
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        self.cuda_device = device
        h = C.c_void_p()
        rc = self._lib.agile_create(config_text(self.cfg).encode(), device, C.byref(h))
        self._ctx = h
        if rc:
            msg = self._lib.agile_last_error(h).decode() if h else ""
            self._lib.agile_destroy(h)
            self._ctx = None
            exc = _lib.CODE_TO_EXC.get(rc, RuntimeError)
            raise exc(f"agile_create: {msg} (rc={rc})")
        if recorder is not None:
            self._check(self._lib.agile_trace_enable(self._ctx, trace_capacity), "trace_enable")
        g = (C.c_uint64 * 11)()
        self._lib.agile_geometry(self._ctx, g, 11)
        (self.num_devices, self.pairs_per_device, self.sq_depth, self.cq_depth, self.num_lines,
         self.ways, self.num_sets, self.engine_warps, self.service_warps, self.infra_ctas,
         fused) = [int(x) for x in g]
        self.launch_mode = "fused" if fused else "split"
        self.engine_copy = self.cfg.engine.copy
        self.devices = [_Device(self, d) for d in range(self.num_devices)]
        self._views = {}

    # ------------------------------------------------------------ plumbing
    def _check(self, rc, what=""):
        _lib.check(self._ctx, rc, what)

    def close(self):
        if getattr(self, "_ctx", None):
            self._views.clear()
            self._lib.agile_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._ctx

    # ------------------------------------------------------------ stores
    def _store_blocks(self, dev):
        p, n = C.c_void_p(), C.c_uint64()
        self._check(self._lib.agile_store_ptr(self._ctx, dev, C.byref(p), C.byref(n)), "store_ptr")
        return int(n.value)

    def attach_store(self, dev: int, num_blocks: int, host_array: np.ndarray | None = None,
                     image_path: str | None = None) -> None:
        ptr = None
        if host_array is not None:
            assert host_array.flags["C_CONTIGUOUS"] and host_array.nbytes >= num_blocks * BLOCK
            ptr = host_array.ctypes.data
            self._views[("owner", dev)] = host_array
        self._views.pop(dev, None)
        self._check(self._lib.agile_store_attach(self._ctx, dev, ptr, num_blocks,
                                                 image_path.encode() if image_path else None), "store_attach")

    def store_view(self, dev: int) -> np.ndarray:
        """Zero-copy uint8 [num_blocks, 4096] view of the pinned store (host side)."""
        v = self._views.get(dev)
        if v is None:
            p, n = C.c_void_p(), C.c_uint64()
            self._check(self._lib.agile_store_ptr(self._ctx, dev, C.byref(p), C.byref(n)), "store_ptr")
            buf = (C.c_uint8 * (int(n.value) * BLOCK)).from_address(p.value)
            v = np.frombuffer(buf, dtype=np.uint8).reshape(int(n.value), BLOCK)
            self._views[dev] = v
        return v

    def fill_store(self, dev: int, seed: int, first_blk: int = 0, nblk: int | None = None,
                   kind: str = "words") -> None:
        """Synthetic contents (oracle/pages.py): kind 'words' = page_words, 'f32' = page_floats."""
        n = self._store_blocks(dev) - first_blk if nblk is None else nblk
        k = {"words": 0, "f32": 1}[kind]
        self._check(self._lib.agile_store_fill(self._ctx, dev, seed, first_blk, n, k), "store_fill")

    def fill_rows(self, dev: int, seed: int, first_blk: int, table: int, row0: int, rows: int, D: int) -> None:
        """Row-keyed embedding table pages (oracle/pages.py row_floats): rows [row0, row0 + rows)
        of `table` from page first_blk on, 4096 / (4 D) rows per page."""
        self._check(self._lib.agile_store_fill_rows(self._ctx, dev, seed, first_blk, table, row0, rows, D),
                    "store_fill_rows")

    def load_image(self, dev: int, path) -> None:
        """BlockStore.load_image (ssd_model.py:84-95) into the attached store; the device's cache
        lines are invalidated and existing store views stay valid."""
        self._check(self._lib.agile_store_load_image(self._ctx, dev, str(path).encode()), "load_image")

    def save_image(self, dev: int, path) -> None:
        self._check(self._lib.agile_store_save_image(self._ctx, dev, str(path).encode()), "save_image")

    # ------------------------------------------------------------ state / counters
    def reset(self, cache=True, queues=True, stats=True) -> None:
        self._check(self._lib.agile_reset(self._ctx, (1 if cache else 0) | (2 if queues else 0)
                                          | (4 if stats else 0)), "reset")

    def stats(self) -> dict:
        out = (C.c_uint64 * len(STAT_NAMES))()
        self._check(self._lib.agile_stats(self._ctx, out, len(STAT_NAMES)), "stats")
        return dict(zip(STAT_NAMES, (int(x) for x in out)))

    @property
    def cache(self):
        return _CacheView(self.stats())

    @property
    def service(self):
        s = self.stats()
        st = ServiceStats(s["completions"], s["windows_rung"], s["drain_entries_rung"],
                          s["barrier_count"], s["barrier_latency_sum"])

        class _S:
            stats = st
        return _S()

    def events(self) -> TraceRecorder:
        """Render the K10 device log into reference trace tuples (appends to ``recorder``)."""
        n = C.c_uint64()
        self._check(self._lib.agile_event_log(self._ctx, None, 0, C.byref(n)), "event_log")
        buf = np.empty(int(n.value) * 64, dtype=np.uint8)
        if n.value:
            self._check(self._lib.agile_event_log(self._ctx, buf.ctypes.data, n.value, C.byref(n)), "event_log")
        rec = TraceRecorder() if self.recorder is None else self.recorder
        return render_event_log(buf.tobytes(), rec)

    def sync(self, stream=None) -> None:
        self._check(self._lib.agile_sync(self._ctx, stream), "sync")

    # ------------------------------------------------------------ workloads
    def run_seq(self, dev, blk, pages: bool = False):
        """Serialized async_read + wait stream; returns (outcome, victims, pages|None).

        outcome: 0 hit, 1 miss, 2 attach; victims: evicted key (dev<<36|blk) or 2**64-1."""
        dev = np.ascontiguousarray(dev, dtype=np.uint32)
        blk = np.ascontiguousarray(blk, dtype=np.uint64)
        n = len(blk)
        out = np.zeros(n, dtype=np.int8)
        vic = np.zeros(n, dtype=np.uint64)
        pg = np.zeros((n, BLOCK), dtype=np.uint8) if pages else None
        self._check(self._lib.agile_run_seq(self._ctx, dev.ctypes.data, blk.ctypes.data, n, out.ctypes.data,
                                            vic.ctypes.data, pg.ctypes.data if pages else None), "run_seq")
        return out, vic, pg

    def run_reads(self, keys, tasks, reads, epochs, async_mode, compute_ns, stream=None, sync=True):
        """CTC epochs; keys: uint64 [epochs, tasks, reads].  Returns dict(t_ns, epoch_t, digest)."""
        import torch
        dev = torch.device("cuda", self.cuda_device)
        k = torch.as_tensor(np.ascontiguousarray(keys, dtype=np.uint64).view(np.int64)).to(dev)
        bufs = torch.empty(tasks * 2 * reads * BLOCK, dtype=torch.uint8, device=dev)
        digest = torch.zeros(tasks, dtype=torch.int64, device=dev)
        et = torch.zeros(epochs + 1, dtype=torch.int64, device=dev)
        st = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
        self._check(self._lib.agile_run_reads(self._ctx, k.data_ptr(), tasks, reads, epochs, int(async_mode),
                                              int(compute_ns), bufs.data_ptr(), digest.data_ptr(),
                                              et.data_ptr(), st), "run_reads")
        if sync:
            self.sync(st)
        e = et.cpu().numpy().astype(np.int64)
        return {"t_ns": int(e[-1] - e[0]), "epoch_t": e, "digest": digest.cpu().numpy().view(np.uint64),
                "bufs": bufs}

    def run_loop(self, conc, warmup_ns, measure_ns, max_per_task=0, write=False):
        """Closed-loop 4 KiB requesters (bench/bandwidth.py:20-42): reads, or writes when `write`."""
        import torch
        dev = torch.device("cuda", self.cuda_device)
        bufs = torch.empty(conc * BLOCK, dtype=torch.uint8, device=dev)
        cnt = torch.zeros(4, dtype=torch.int64, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        self._check(self._lib.agile_run_loop_rw(self._ctx, conc, int(warmup_ns), int(measure_ns), int(max_per_task),
                                                bufs.data_ptr(), cnt.data_ptr(), 1 if write else 0, st), "run_loop")
        self.sync(st)
        c = cnt.cpu().numpy()
        return {"completions": int(c[0]), "window_ns": int(c[2] - c[1])}

    def write_blocks(self, dev, blk, pages: np.ndarray) -> None:
        """async_write + wait of whole blocks (AgileApi.async_write, gpu_api.py:192-227): each
        lands in its cache line and is written through to the device store."""
        dev = np.ascontiguousarray(dev, dtype=np.uint32)
        blk = np.ascontiguousarray(blk, dtype=np.uint64)
        pages = np.ascontiguousarray(pages, dtype=np.uint8).reshape(len(blk), BLOCK)
        self._check(self._lib.agile_write_blocks(self._ctx, dev.ctypes.data, blk.ctypes.data, len(blk),
                                                 pages.ctypes.data), "write_blocks")

    def evict_blocks(self, dev, blk) -> np.ndarray:
        """SoftwareCache.evict per block: 0 RESET, 1 DEFERRED, 2 not resident, 3 WRITEBACK_STARTED."""
        dev = np.ascontiguousarray(dev, dtype=np.uint32)
        blk = np.ascontiguousarray(blk, dtype=np.uint64)
        out = np.zeros(len(blk), dtype=np.int8)
        self._check(self._lib.agile_evict_blocks(self._ctx, dev.ctypes.data, blk.ctypes.data, len(blk),
                                                 out.ctypes.data), "evict_blocks")
        return out

    def flush(self) -> int:
        """SoftwareCache.flush (software_cache.py:283-298): write back every MODIFIED line."""
        n = C.c_uint64(0)
        self._check(self._lib.agile_flush(self._ctx, C.byref(n)), "flush")
        return int(n.value)

    def lock_cycle_demo(self, n: int, mode: int = 0) -> None:
        """Planted lock-order bug (mode 0: ring of n warps, 1: a warp re-taking its lock); raises
        LockCycle when debug_locks reports the wait-for cycle (lock_chain.py DeadlockDetector)."""
        self._check(self._lib.agile_lock_cycle_demo(self._ctx, n, mode), "lock_cycle_demo")

    def buffer_busy_demo(self, write: bool = False) -> None:
        """Re-use a buffer whose transfer is pending (raises BufferBusy, gpu_api.py:132-137)."""
        self._check(self._lib.agile_buffer_busy_demo(self._ctx, int(write)), "buffer_busy_demo")

    def share_live(self) -> int:
        """ShareTable.live_entries (share_table.py:198-199); 0 when the table is disabled."""
        n = C.c_uint64(0)
        self._check(self._lib.agile_share_live(self._ctx, C.byref(n)), "share_live")
        return int(n.value)

    def run_coherence(self, op, blk, think):
        """The reference's coherence workload (tests/test_coherence.py:27-60) on the device:
        op/blk/think are [tasks][ops] arrays (op 0 read, 1 write).  Returns (seen [tasks][ops]
        observed prefixes, lines flushed at the end)."""
        op = np.ascontiguousarray(op, dtype=np.uint8)
        tasks, ops = op.shape
        blk = np.ascontiguousarray(blk, dtype=np.uint32).reshape(tasks, ops)
        think = np.ascontiguousarray(think, dtype=np.uint32).reshape(tasks, ops)
        seen = np.zeros((tasks, ops), dtype=np.uint64)
        fl = C.c_uint64(0)
        self._check(self._lib.agile_run_coherence(self._ctx, op.ctypes.data, blk.ctypes.data, think.ctypes.data,
                                                  tasks, ops, seen.ctypes.data, C.byref(fl)), "run_coherence")
        return seen, int(fl.value)

    def set_engine_copy(self, mode: str) -> None:
        """engine.copy of later runs: 'registers' | 'bulk'."""
        self._check(self._lib.agile_set_engine_copy(self._ctx, {"registers": 0, "bulk": 1}[mode]), "set_engine_copy")
        self.engine_copy = mode

    def set_launch_mode(self, mode: str) -> None:
        """'split' | 'fused' | 'solo' (split launch whose user grid may run alone) | 'users' (no
        infra grid: profiling of all-hit replays under a kernel-serialising tool)."""
        code = {"split": 0, "fused": 1, "solo": 2, "users": 3}[mode]
        self._check(self._lib.agile_set_launch_mode(self._ctx, code), "set_launch_mode")
        self.launch_mode = "fused" if mode == "fused" else "split"

    def array_get(self, dev, idx, elem_size: int = 4):
        """AgileApi.array_get (gpu_api.py:250-278): synchronous element read, the device viewed as a
        little-endian array of elem_size-byte elements.  Scalars return an int; arrays of indices
        (with a scalar or per-element dev) return a list of ints (elem_size > 8) or a uint64 array."""
        if elem_size <= 0 or BLOCK % elem_size:
            raise ValueError("element size must divide the block size")
        scalar = np.isscalar(idx)
        idx = np.atleast_1d(np.ascontiguousarray(idx, dtype=np.uint64))
        dev = np.ascontiguousarray(np.broadcast_to(np.asarray(dev, dtype=np.uint32), idx.shape))
        out = np.zeros((len(idx), elem_size), dtype=np.uint8)
        self._check(self._lib.agile_array_get(self._ctx, dev.ctypes.data, idx.ctypes.data, len(idx), elem_size,
                                              out.ctypes.data), "array_get")
        vals = [int.from_bytes(row.tobytes(), "little") for row in out]
        if scalar:
            return vals[0]
        return np.array(vals, dtype=np.uint64) if elem_size <= 8 else vals

    def run_gather(self, keys, tasks, epochs, gathers, async_mode, compute_ns):
        import torch
        dev = torch.device("cuda", self.cuda_device)
        k = torch.as_tensor(np.ascontiguousarray(keys, dtype=np.uint64).view(np.int64)).to(dev)
        vals = torch.zeros(tasks * epochs * gathers, dtype=torch.int32, device=dev)
        et = torch.zeros(2, dtype=torch.int64, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        self._check(self._lib.agile_run_gather(self._ctx, k.data_ptr(), tasks, epochs, gathers, int(async_mode),
                                               int(compute_ns), vals.data_ptr(), et.data_ptr(), st), "run_gather")
        self.sync(st)
        e = et.cpu().numpy()
        return {"t_ns": int(e[1] - e[0]), "values": vals.cpu().numpy().view(np.uint32)}

    def embbag(self, idx, table_key0, table_rows, out, counters, prefetch_distance=1, stream=None,
               out_b_stride=0, out_t_stride=0, user_ctas=0):
        """Device-tensor embedding-bag (sum pooling) through the page cache; async launch.
        user_ctas bounds the user CTAs of the launch (0 = every resident slot)."""
        import torch
        if not idx.is_contiguous() or not out.is_contiguous():
            raise ValueError("embbag: idx and out must be contiguous")
        B, T, L = idx.shape
        D = out.shape[-1]
        st = stream if stream is not None else torch.cuda.current_stream(idx.device).cuda_stream
        self._check(self._lib.agile_embbag_ctas(self._ctx, idx.data_ptr(), table_key0.data_ptr(),
                                                table_rows.data_ptr(), out.data_ptr(), counters.data_ptr(), B, T, L,
                                                D, out_b_stride, out_t_stride, prefetch_distance, user_ctas, st),
                    "embbag")

    def embbag_sharded(self, idx, tables, out, counters, D, offsets=None, prefetch_distance=0, user_ctas=0,
                       prefetch_only=False, stream=None, B=None, L=None):
        """Sharded / variable-length embedding-bag (agile_embbag_sharded): `tables` is a device
        tensor holding one agile_table_shard (40 B, bench.dlrm.TAB_DTYPE) per table of the launch;
        `out` is a device buffer whose rows (one per sample) receive each table's pooled vector at
        its out_offset — fp32, or fp64 partial sums for row-wise pieces.  idx [B, T, L] int64, or
        with offsets [B*T + 1] a flat index array (pass B)."""
        import torch
        for name, t in (("idx", idx), ("tables", tables), ("out", out), ("offsets", offsets)):
            if t is not None and not t.is_contiguous():
                raise ValueError(f"embbag_sharded: {name} must be contiguous")
        T = tables.numel() * tables.element_size() // 40
        if offsets is None:
            B, _, L = idx.shape
            off_ptr = 0
        else:
            L = 0
            off_ptr = offsets.data_ptr()
        row_bytes = 0 if out is None else out.numel() * out.element_size() // max(1, B)
        st = stream if stream is not None else torch.cuda.current_stream(idx.device).cuda_stream
        self._check(self._lib.agile_embbag_sharded(self._ctx, idx.data_ptr(), off_ptr, tables.data_ptr(),
                                                   0 if out is None else out.data_ptr(), row_bytes,
                                                   counters.data_ptr(), B, T, L, D, prefetch_distance, user_ctas,
                                                   1 if prefetch_only else 0, st), "embbag_sharded")

    def embbag_prefetch(self, idx, table_key0, table_rows, D, counters, user_ctas=0, stream=None):
        """Pull every page of the batch into the cache (async launch on `stream`)."""
        import torch
        B, T, L = idx.shape
        st = stream if stream is not None else torch.cuda.current_stream(idx.device).cuda_stream
        self._check(self._lib.agile_embbag_prefetch(self._ctx, idx.data_ptr(), table_key0.data_ptr(),
                                                    table_rows.data_ptr(), counters.data_ptr(), B, T, L, D,
                                                    user_ctas, st), "embbag_prefetch")

    def embbag_host(self, idx: np.ndarray, table_key0: np.ndarray, table_rows: np.ndarray, D: int,
                    prefetch_distance=1, out: np.ndarray | None = None):
        """Host-buffer embedding-bag through the C-ABI (H2D + kernel + D2H inside)."""
        B, T, L = idx.shape
        if out is None:
            out = np.empty((B, T, D), dtype=np.float32)
        cnt = np.zeros(2, dtype=np.uint64)
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        k0 = np.ascontiguousarray(table_key0, dtype=np.uint64)
        rows = np.ascontiguousarray(table_rows, dtype=np.int64)
        self._check(self._lib.agile_embbag_host(self._ctx, idx.ctypes.data, k0.ctypes.data, rows.ctypes.data,
                                                out.ctypes.data, cnt.ctypes.data, B, T, L, D, prefetch_distance),
                    "embbag_host")
        return out, cnt

    def embbag_host_submit(self, idx: np.ndarray, table_key0: np.ndarray, table_rows: np.ndarray, D: int,
                           out: np.ndarray, counters: np.ndarray, slot: int, prefetch_distance=0):
        """Asynchronous host-buffer embedding-bag on staging slot 0/1 (copies of one slot overlap
        the other's run); buffers must stay alive (and should be pinned) until embbag_host_wait."""
        B, T, L = idx.shape
        self._check(self._lib.agile_embbag_host_submit(self._ctx, idx.ctypes.data, table_key0.ctypes.data,
                                                       table_rows.ctypes.data, out.ctypes.data,
                                                       counters.ctypes.data, B, T, L, D, prefetch_distance,
                                                       slot), "embbag_host_submit")

    def embbag_host_wait(self, slot: int) -> None:
        self._check(self._lib.agile_embbag_host_wait(self._ctx, slot), "embbag_host_wait")

    def bfs(self, row_ptr, V, source, col_key0, level, prefetch_distance=0, stream=None):
        """Whole BFS over a paged CSR (one fused launch per level); returns the stats dict."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(row_ptr.device).cuda_stream
        stats = np.zeros(4, dtype=np.uint64)
        self._check(self._lib.agile_bfs(self._ctx, row_ptr.data_ptr(), V, source, col_key0, level.data_ptr(),
                                        prefetch_distance, stats.ctypes.data, st), "bfs")
        return {"levels": int(stats[0]), "edges": int(stats[1]), "page_misses": int(stats[2]),
                "ms": int(stats[3]) / 1e6}

    def spmv(self, row_ptr, V, E, col_key0, val_key0, x, y, alpha=1.0, beta=0.0, prefetch_distance=0,
             counters=None, stream=None):
        """y = alpha * A x + beta over a paged CSR (async launch)."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(row_ptr.device).cuda_stream
        if counters is None:
            counters = torch.zeros(2, dtype=torch.int64, device=row_ptr.device)
        vk = (1 << 64) - 1 if val_key0 is None else val_key0
        self._check(self._lib.agile_spmv(self._ctx, row_ptr.data_ptr(), V, E, col_key0, vk, x.data_ptr(),
                                         y.data_ptr(), float(alpha), float(beta), prefetch_distance,
                                         counters.data_ptr(), st), "spmv")
        return counters

    def spmv_rows(self, row_ptr, n_rows, e_end, x_len, col_key0, val_key0, x, y, alpha=1.0, beta=0.0,
                  prefetch_distance=0, counters=None, stream=None):
        """SpMV over the rows of a 1D vertex partition (agile_spmv_rows): row_ptr[0] may be > 0
        (positions before it belong to the previous partition); x has x_len entries."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(row_ptr.device).cuda_stream
        if counters is None:
            counters = torch.zeros(2, dtype=torch.int64, device=row_ptr.device)
        vk = (1 << 64) - 1 if val_key0 is None else val_key0
        self._check(self._lib.agile_spmv_rows(self._ctx, row_ptr.data_ptr(), n_rows, e_end, x_len, col_key0, vk,
                                              x.data_ptr(), y.data_ptr(), float(alpha), float(beta),
                                              prefetch_distance, counters.data_ptr(), st), "spmv_rows")
        return counters

    def bfs_level(self, row_ptr, v0, frontier, visited, next_bits, level, cur, col_key0, prefetch_distance=0,
                  counters=None, stream=None):
        """One BFS level over the owned frontier of a 1D vertex partition (agile_bfs_level)."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(row_ptr.device).cuda_stream
        n = frontier.numel()
        self._check(self._lib.agile_bfs_level(self._ctx, row_ptr.data_ptr(), v0, frontier.data_ptr() if n else 0, n,
                                              visited.data_ptr(), next_bits.data_ptr(), level.data_ptr(), cur,
                                              col_key0, prefetch_distance, counters.data_ptr(), st), "bfs_level")

    def embbag_grid(self):
        u, i = C.c_uint32(), C.c_uint32()
        self._check(self._lib.agile_embbag_grid(self._ctx, C.byref(u), C.byref(i)), "embbag_grid")
        return int(u.value), int(i.value)
