"""B200-native PystachIO hot path (arxiv 2512.02862): storage-resident OLAP execution on sm_100a.

Python face of the C-ABI in ``include/psg.h`` (ctypes over the in-tree ``libpsg.so``). The
function names and argument meanings mirror the reference's pybind11 module
(``/root/reference/proj/python/bindings.cpp:98-231``): ``tmin``, ``write_table``, ``inspect``,
``scan``, ``gen_workload`` and — replacing ``run_plan_sim`` — ``run_plan`` which executes
``execute_plan`` on the GPU. Operator adapters (``filter``, ``partition``, ``hash_join``) mirror
``ops.hpp:35-83``. There is no CPU fallback: without the built extension or a CUDA device every
compute call raises.
"""
from __future__ import annotations

import ctypes
import json
import math
import os

import numpy as np

__all__ = ["Context", "PsgError", "tmin", "write_table", "inspect", "scan", "gen_workload", "run_plan",
           "filter", "partition", "hash_join", "lib", "MODES", "STATUS"]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libpsg.so")

MODES = {"blocking": 0, "fastio": 1, "combined": 2, "overlapped": 3}
STATUS = {0: "OK", 1: "UnknownColumn", 2: "MemoryExceeded", 3: "StreamClosed", 4: "IoFailure", 5: "CorruptFooter",
          6: "CollectiveOrderViolation", 7: "PeerDisconnected", 8: "ChecksumMismatch", 9: "InvalidInput",
          10: "InfeasibleBudget", 11: "MalformedTrace", 12: "EmptyTrace", 100: "CudaError", 101: "NcclError",
          102: "InternalError"}
EXPORTS = ["psg_abi_version", "psg_last_error", "psg_ctx_create", "psg_comm_unique_id", "psg_ctx_init_comm",
           "psg_ctx_set_ingest", "psg_ctx_set_semijoin", "psg_ctx_set_fused_shuffle", "psg_ctx_destroy", "psg_execute_plan",
           "psg_execute_local", "psg_stage_plan",
           "psg_execute_staged", "psg_staged_free", "psg_result_shape", "psg_result_field", "psg_result_data",
           "psg_result_stats", "psg_result_free", "psg_filter", "psg_partition", "psg_hash_join", "psg_hashtable_build",
           "psg_hashtable_shape", "psg_hashtable_row", "psg_hashtable_lookup", "psg_hashtable_probe", "psg_hashtable_free",
           "psg_concat", "psg_codec_decompress", "psg_psto_write",
           "psg_psto_inspect", "psg_gen_tpch", "psg_gen_synthetic", "psg_jit_selftest", "psg_tmin",
           "psg_plan_resolve", "psg_result_checksum", "psg_ingest_probe",
           "psg_shuffle_plan", "psg_pack_plan", "psg_partition_of", "psg_join_schedule", "psg_run_synthetic_join"]


class PsgError(RuntimeError):
    """Engine error; ``kind`` names the reference exception class (errors.hpp:21-87)."""

    def __init__(self, code, msg):
        self.code = code
        self.kind = STATUS.get(code, "Error%d" % code)
        super().__init__("%s: %s" % (self.kind, msg))


class Stats(ctypes.Structure):
    _fields_ = [("runtime_s", ctypes.c_double), ("storage_phase_s", ctypes.c_double),
                ("network_phase_s", ctypes.c_double), ("peak_bytes", ctypes.c_uint64),
                ("bytes_received", ctypes.c_uint64), ("ingest_bytes", ctypes.c_uint64),
                ("result_bytes", ctypes.c_uint64), ("kernel_launches", ctypes.c_uint64),
                ("waves", ctypes.c_uint64), ("probe_kernel_ms", ctypes.c_double),
                ("probe_kernel_launches", ctypes.c_uint64), ("probe_kernel_bytes", ctypes.c_uint64),
                ("device_ms", ctypes.c_double), ("result_rows", ctypes.c_uint64), ("io_wait_s", ctypes.c_double),
                ("jit_compiles", ctypes.c_uint64), ("h2d_bytes", ctypes.c_uint64),
                ("agg_table", ctypes.c_uint64), ("bytes_sent", ctypes.c_uint64), ("exchange_ms", ctypes.c_double),
                ("bucket_overflow", ctypes.c_uint64), ("shuffle_fused", ctypes.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


JOIN_VARIANTS = {"blocking": 0, "blocking-opt": 1, "chunking": 2, "deferred": 3}


class JoinSpec(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int), ("stream_count", ctypes.c_int), ("chunk_rows", ctypes.c_uint64)]


class JoinWorkload(ctypes.Structure):
    _fields_ = [("build_rows", ctypes.c_uint64), ("probe_rows", ctypes.c_uint64), ("payload_cols", ctypes.c_int),
                ("hit_ratio", ctypes.c_double), ("seed", ctypes.c_uint64)]


class JoinStats(ctypes.Structure):
    _fields_ = [("runtime_s", ctypes.c_double), ("device_ms", ctypes.c_double), ("result_rows", ctypes.c_uint64),
                ("bytes_received", ctypes.c_uint64), ("left_waves", ctypes.c_uint64), ("right_waves", ctypes.c_uint64),
                ("host_syncs", ctypes.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Batch(ctypes.Structure):
    _fields_ = [("ncols", ctypes.c_uint32), ("nrows", ctypes.c_uint64), ("names", ctypes.POINTER(ctypes.c_char_p)),
                ("types", ctypes.POINTER(ctypes.c_uint8)), ("cols", ctypes.POINTER(ctypes.POINTER(ctypes.c_uint64)))]


class Atom(ctypes.Structure):
    _fields_ = [("column", ctypes.c_char_p), ("op", ctypes.c_char_p), ("literal_is_float", ctypes.c_int),
                ("literal_i", ctypes.c_int64), ("literal_f", ctypes.c_double)]


_lib = None


def lib():
    """The loaded ``libpsg.so`` (raises if the extension was not built: no fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError("libpsg.so not built: run `python -m paper_2512_02862_b200.build` "
                              "(the B200 path has no CPU fallback)")
        L = ctypes.CDLL(_LIB_PATH)
        vp, u64, i32, c = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_char_p
        P = ctypes.POINTER
        sig = {
            "psg_abi_version": ([], i32), "psg_last_error": ([], c),
            "psg_ctx_create": ([i32, i32, i32, P(vp)], i32), "psg_comm_unique_id": ([vp], i32),
            "psg_ctx_init_comm": ([vp, vp], i32), "psg_ctx_set_ingest": ([vp, i32, u64, i32], i32),
            "psg_ctx_set_semijoin": ([vp, i32], i32), "psg_ctx_set_fused_shuffle": ([vp, i32], i32),
            "psg_ctx_destroy": ([vp], None),
            "psg_execute_plan": ([vp, c, c, i32, P(vp)], i32), "psg_stage_plan": ([vp, c, c, P(vp)], i32),
            "psg_execute_local": ([vp, c, c, i32, P(vp)], i32),
            "psg_execute_staged": ([vp, vp, i32, P(vp), P(Stats)], i32), "psg_staged_free": ([vp], None),
            "psg_result_shape": ([vp, P(u64), P(ctypes.c_uint32)], i32),
            "psg_result_field": ([vp, ctypes.c_uint32, P(c), P(i32)], i32),
            "psg_result_data": ([vp], P(u64)), "psg_result_stats": ([vp, P(Stats)], i32),
            "psg_result_free": ([vp], None),
            "psg_filter": ([vp, P(Batch), P(Atom), ctypes.c_uint32, P(vp)], i32),
            "psg_partition": ([vp, P(Batch), c, ctypes.c_uint32, i32, P(vp), P(u64)], i32),
            "psg_hash_join": ([vp, P(Batch), c, P(Batch), c, P(vp)], i32),
            "psg_hashtable_build": ([vp, P(Batch), ctypes.c_uint32, c, i32, P(vp)], i32),
            "psg_hashtable_shape": ([vp, P(u64), P(ctypes.c_uint32)], i32),
            "psg_hashtable_row": ([vp, c, u64, P(ctypes.c_int64), P(u64)], i32),
            "psg_hashtable_lookup": ([vp, vp, P(ctypes.c_int64), u64, P(u64), P(u64), u64, P(u64)], i32),
            "psg_hashtable_probe": ([vp, vp, P(Batch), c, P(vp)], i32),
            "psg_hashtable_free": ([vp], None),
            "psg_concat": ([vp, P(Batch), ctypes.c_uint32, P(vp)], i32),
            "psg_codec_decompress": ([vp, i32, u64, P(vp), P(u64), P(vp), P(u64)], i32),
            "psg_psto_write": ([c, P(Batch), u64, i32, P(u64)], i32),
            "psg_psto_inspect": ([c, P(u64), P(ctypes.c_uint32), P(u64), P(i32)], i32),
            "psg_gen_tpch": ([c, ctypes.c_double, i32, i32, u64, i32, u64, i32], i32),
            "psg_gen_synthetic": ([c, i32, i32, u64, i32, u64, u64, u64, i32, ctypes.c_double], i32),
            "psg_tmin": ([u64, ctypes.c_double, u64, ctypes.c_double], ctypes.c_double),
            "psg_jit_selftest": ([ctypes.c_char_p, ctypes.c_size_t], i32),
            "psg_ingest_probe": ([vp, c, c, P(Stats)], i32),
            "psg_join_schedule": ([i32, i32, i32, i32, P(ctypes.c_int32), ctypes.c_size_t, P(ctypes.c_size_t)], i32),
            "psg_run_synthetic_join": ([vp, P(JoinSpec), P(JoinWorkload), i32, P(JoinStats), P(vp)], i32),
            "psg_shuffle_plan": ([P(u64), i32, i32, P(u64), P(u64), P(u64), P(u64)], i32),
            "psg_pack_plan": ([P(ctypes.c_int64), P(ctypes.c_int64), i32, P(ctypes.c_int64), P(i32), P(u64), P(i32)], i32),
            "psg_partition_of": ([P(ctypes.c_int64), u64, ctypes.c_uint32, P(ctypes.c_uint32)], i32),
            "psg_result_checksum": ([vp, P(u64), P(u64), ctypes.c_uint32], i32),
            "psg_plan_resolve": ([c, c, i32, i32, ctypes.c_char_p, ctypes.c_size_t, P(ctypes.c_size_t)], i32),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise PsgError(rc, lib().psg_last_error().decode(errors="replace"))


def join_schedule(variant, stream_count, left_waves, right_waves):
    """The join schedule [(phase, stream, wave)] (PlanStep list of make_plan, join.cpp:126-134)."""
    n = ctypes.c_size_t()
    v = JOIN_VARIANTS[variant] if isinstance(variant, str) else variant
    _check(lib().psg_join_schedule(v, stream_count, left_waves, right_waves, None, 0, ctypes.byref(n)))
    buf = (ctypes.c_int32 * (3 * max(n.value, 1)))()
    _check(lib().psg_join_schedule(v, stream_count, left_waves, right_waves, buf, n.value, ctypes.byref(n)))
    return [[buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]] for i in range(n.value)]


def shuffle_plan(matrix, me):
    """(send_off, recv_off, send_rows, recv_rows) of rank `me` from the all-gathered n x n count
    matrix [src][dst] - the engine's own host function (csrc/shuffle_plan.cpp)."""
    m = np.ascontiguousarray(matrix, dtype=np.uint64)
    n = m.shape[0]
    so, ro = np.zeros(n, np.uint64), np.zeros(n, np.uint64)
    sr, rr = ctypes.c_uint64(), ctypes.c_uint64()
    P = ctypes.POINTER(ctypes.c_uint64)
    _check(lib().psg_shuffle_plan(m.ctypes.data_as(P), n, me, so.ctypes.data_as(P), ro.ctypes.data_as(P),
                                  ctypes.byref(sr), ctypes.byref(rr)))
    return so, ro, sr.value, rr.value


def pack_plan(lo, hi):
    """One-word shuffle-row layout {fits, min, shift, mask} from all-reduced bounds."""
    lo = np.ascontiguousarray(lo, dtype=np.int64)
    hi = np.ascontiguousarray(hi, dtype=np.int64)
    k = len(lo)
    mn, sh, mk = np.zeros(k, np.int64), np.zeros(k, np.int32), np.zeros(k, np.uint64)
    fits = ctypes.c_int()
    I64 = ctypes.POINTER(ctypes.c_int64)
    _check(lib().psg_pack_plan(lo.ctypes.data_as(I64), hi.ctypes.data_as(I64), k, mn.ctypes.data_as(I64),
                               sh.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                               mk.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), ctypes.byref(fits)))
    return {"fits": bool(fits.value), "min": mn, "shift": sh, "mask": mk}


def partition_of(keys, nparts):
    """Destination rank of each key (hashing.hpp:35-37), host evaluation."""
    k = np.ascontiguousarray(keys, dtype=np.int64)
    out = np.zeros(len(k), np.uint32)
    _check(lib().psg_partition_of(k.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), len(k), nparts,
                                  out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))))
    return out


def resolve_plan(plan, data_root, node=0, nodes=1):
    """Host-only plan parse + validation (QueryPlan::from_json_text, pipeline.cpp:108-156): the
    resolved scans {"scans": [{"table", "replicated", "paths"}], "shuffle": id | None}."""
    text = (plan if isinstance(plan, str) else json.dumps(plan)).encode()
    need = ctypes.c_size_t(0)
    _check(lib().psg_plan_resolve(text, data_root.encode(), node, nodes, None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check(lib().psg_plan_resolve(text, data_root.encode(), node, nodes, buf, need.value, None))
    return json.loads(buf.value.decode())


# ------------------------------------------------------------------------------ batches
def _make_batch(columns: dict, types: dict | None = None):
    """dict name -> sequence/ndarray. int -> Int64, float -> Float64 (raw 8-byte words)."""
    names, tys, arrs = [], [], []
    n = None
    for name, vals in columns.items():
        a = np.asarray(vals)
        t = (types or {}).get(name)
        if t is None:
            t = 1 if a.dtype.kind == "f" else 0
        if a.dtype == np.uint64:  # already raw 8-byte words
            a = np.ascontiguousarray(a)
        elif t == 1:
            a = np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)
        else:
            a = np.ascontiguousarray(a.astype(np.int64, copy=False)).view(np.uint64)
        if n is None:
            n = len(a)
        elif len(a) != n:
            raise PsgError(9, "ragged batch: column row counts differ")
        names.append(name.encode())
        tys.append(t)
        arrs.append(a)
    nc = len(names)
    b = Batch()
    b.ncols = nc
    b.nrows = n or 0
    b._names = (ctypes.c_char_p * max(nc, 1))(*names)
    b._types = (ctypes.c_uint8 * max(nc, 1))(*tys)
    b._arrs = arrs
    b._cols = (ctypes.POINTER(ctypes.c_uint64) * max(nc, 1))(
        *[a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)) for a in arrs])
    b.names = ctypes.cast(b._names, ctypes.POINTER(ctypes.c_char_p))
    b.types = ctypes.cast(b._types, ctypes.POINTER(ctypes.c_uint8))
    b.cols = ctypes.cast(b._cols, ctypes.POINTER(ctypes.POINTER(ctypes.c_uint64)))
    return b


class _Owner:
    """Owns a psg_result handle; freed as soon as the last Result/ndarray view referencing it dies
    (no reference cycle, so the engine's pinned result block returns to its cache immediately)."""

    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        try:
            if self.h is not None:
                lib().psg_result_free(self.h)
                self.h = None
        except Exception:
            pass


class _View:
    """Array-interface wrapper whose lifetime pins the result handle (numpy keeps it as .base)."""

    def __init__(self, owner, ptr, n):
        self._owner = owner
        self.__array_interface__ = {"shape": (n,), "typestr": "<u8", "version": 3,
                                    "data": (ctypes.cast(ptr, ctypes.c_void_p).value, False)}


class Result:
    """PipelineResult (pipeline.hpp:138-149): schema + rows of raw u64 words (row-major ndarray)."""

    def __init__(self, handle):
        L = lib()
        n, k = ctypes.c_uint64(), ctypes.c_uint32()
        _check(L.psg_result_shape(handle, ctypes.byref(n), ctypes.byref(k)))
        self.schema = []
        for i in range(k.value):
            nm, ty = ctypes.c_char_p(), ctypes.c_int()
            _check(L.psg_result_field(handle, i, ctypes.byref(nm), ctypes.byref(ty)))
            self.schema.append((nm.value.decode(), "float64" if ty.value == 1 else "int64"))
        cnt = n.value * k.value
        ptr = L.psg_result_data(handle)
        st = Stats()
        _check(L.psg_result_stats(handle, ctypes.byref(st)))
        self.stats = st.as_dict()
        if cnt:
            # zero-copy view of the engine's (pinned) result rows
            self._owner = _Owner(handle)
            self.rows = np.asarray(_View(self._owner, ptr, cnt)).reshape(n.value, k.value)
        else:
            self.rows = np.zeros((n.value, k.value), np.uint64)
            L.psg_result_free(handle)

    def checksum(self):
        """{"rows", "rowhash", "colsums"}: rowhash = sum over rows of FNV-1a64 of the row's words
        (mod 2^64, additive over ranks), the reference harness's result checksum."""
        k = len(self.schema)
        if self.rows.shape[0] == 0:
            return {"rows": 0, "rowhash": "%016x" % 0, "colsums": ["0"] * k}
        h = ctypes.c_uint64()
        cs = (ctypes.c_uint64 * max(k, 1))()
        _check(lib().psg_result_checksum(self._owner.h, ctypes.byref(h), cs, k))
        return {"rows": int(self.rows.shape[0]), "rowhash": "%016x" % h.value, "colsums": [str(cs[i]) for i in range(k)]}

    def column(self, name):
        i = [n for n, _t in self.schema].index(name)
        col = self.rows[:, i]
        return col.view(np.float64) if self.schema[i][1] == "float64" else col.view(np.int64)

    def to_dict(self):
        return {n: self.column(n).tolist() for n, _t in self.schema}


class Context:
    """One GPU / one rank (ExecEnv + Fabric + DeviceManager, exec.hpp:84-92)."""

    def __init__(self, device=0, rank=0, nranks=1, nccl_id: bytes | None = None):
        L = lib()
        h = ctypes.c_void_p()
        _check(L.psg_ctx_create(device, rank, nranks, ctypes.byref(h)))
        self._h = h
        self.device, self.rank, self.nranks = device, rank, nranks
        if nranks > 1:
            if nccl_id is None:
                raise PsgError(9, "nranks > 1 needs the NCCL unique id from rank 0 (Context.unique_id())")
            buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            _check(L.psg_ctx_init_comm(self._h, buf))

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(lib().psg_comm_unique_id(buf))
        return buf.raw

    def set_ingest(self, io_threads=-1, batch_bytes=0, pinned_slots=-1):
        _check(lib().psg_ctx_set_ingest(self._h, io_threads, batch_bytes, pinned_slots))

    def set_semijoin(self, enabled: bool):
        _check(lib().psg_ctx_set_semijoin(self._h, 1 if enabled else 0))

    def set_fused_shuffle(self, enabled: bool):
        """nranks > 1: fused NVLink build/probe (True) or the NCCL partition/send/recv path (False)."""
        _check(lib().psg_ctx_set_fused_shuffle(self._h, 1 if enabled else 0))

    def execute_plan(self, plan, data_root, mode="overlapped") -> Result:
        text = plan if isinstance(plan, str) else json.dumps(plan)
        out = ctypes.c_void_p()
        _check(lib().psg_execute_plan(self._h, text.encode(), data_root.encode(), MODES[mode], ctypes.byref(out)))
        return Result(out)

    def execute_local(self, plan, data_root, mode="overlapped") -> Result:
        """Plans without a shuffled join (scan -> replicated joins -> global aggregate, the Q6
        analog); one partial row [rows, sums...] for this rank's node. Extension: the reference's
        execute_plan rejects such plans (pipeline.cpp:334-335)."""
        text = plan if isinstance(plan, str) else json.dumps(plan)
        out = ctypes.c_void_p()
        _check(lib().psg_execute_local(self._h, text.encode(), data_root.encode(), MODES[mode], ctypes.byref(out)))
        return Result(out)

    def run_synthetic_join(self, variant="deferred", stream_count=2, chunk_rows=32 * 1024, build_rows=120_000,
                           probe_rows=320_000, payload_cols=3, hit_ratio=0.5, seed=42, collect_rows=True):
        """run_join (join.cpp) over this rank's slice of the synthetic join workload
        (SyntheticJoinSpec, workload.hpp:27-33). Returns (stats dict, Result or None)."""
        spec = JoinSpec(JOIN_VARIANTS[variant] if isinstance(variant, str) else variant, stream_count, chunk_rows)
        wl = JoinWorkload(build_rows, probe_rows, payload_cols, hit_ratio, seed)
        st = JoinStats()
        out = ctypes.c_void_p()
        _check(lib().psg_run_synthetic_join(self._h, ctypes.byref(spec), ctypes.byref(wl), 1 if collect_rows else 0,
                                            ctypes.byref(st), ctypes.byref(out) if collect_rows else None))
        return st.as_dict(), (Result(out) if collect_rows else None)

    def ingest_probe(self, plan, data_root) -> dict:
        """The plan's storage -> pinned -> HBM ingest alone (same session as execute_plan, no query
        kernels): stats dict with runtime_s / h2d_bytes - the e2e roofline's ingest term."""
        text = plan if isinstance(plan, str) else json.dumps(plan)
        st = Stats()
        _check(lib().psg_ingest_probe(self._h, text.encode(), data_root.encode(), ctypes.byref(st)))
        return st.as_dict()

    def stage_plan(self, plan, data_root):
        text = plan if isinstance(plan, str) else json.dumps(plan)
        out = ctypes.c_void_p()
        _check(lib().psg_stage_plan(self._h, text.encode(), data_root.encode(), ctypes.byref(out)))
        return Staged(self, out)

    def close(self):
        if getattr(self, "_h", None):
            lib().psg_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class Staged:
    """Plan inputs resident in HBM (psg_stage_plan); run() executes without host I/O."""

    def __init__(self, ctx, handle):
        self.ctx, self._h = ctx, handle

    def run(self, mode="overlapped", want_rows=True):
        out = ctypes.c_void_p()
        st = Stats()
        _check(lib().psg_execute_staged(self.ctx._h, self._h, MODES[mode], ctypes.byref(out) if want_rows else None,
                                        ctypes.byref(st)))
        return Result(out) if want_rows else st.as_dict()

    def free(self):
        if self._h:
            lib().psg_staged_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


_default_ctx = None


def _ctx():
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# --------------------------------------------------------------- reference-shaped functions
def jit_selftest():
    """NVRTC-compile representative fused-scan programs for sm_100a (no GPU needed)."""
    buf = ctypes.create_string_buffer(1 << 16)
    n = lib().psg_jit_selftest(buf, len(buf))
    return n, buf.value.decode(errors="replace")


def tmin(ssd_read_size_agg, ssd_read_bw_agg, net_recv_size_node, net_bw):
    """Eq. 1 (bench.cpp:35-40): max(storage read time, per-node network receive time), seconds."""
    v = lib().psg_tmin(int(ssd_read_size_agg), float(ssd_read_bw_agg), int(net_recv_size_node), float(net_bw))
    if math.isnan(v):
        raise PsgError(9, lib().psg_last_error().decode())
    return v


def write_table(path, columns: dict, row_group_rows=65536, codec="identity"):
    """Writes a PSTO table (TableWriter, psto.cpp:144-229); returns the row-group count."""
    b = _make_batch(columns)
    g = ctypes.c_uint64()
    _check(lib().psg_psto_write(path.encode(), ctypes.byref(b), int(row_group_rows), 1 if codec == "block" else 0,
                                ctypes.byref(g)))
    return g.value


def _footer_schema(path):
    import struct
    with open(path, "rb") as f:
        f.seek(-12, 2)
        flen = struct.unpack("<Q", f.read(8))[0]
        f.seek(-12 - flen, 2)
        foot = f.read(flen)
    off = 5
    (nc,) = struct.unpack_from("<I", foot, off)
    off += 4
    schema = []
    for _ in range(nc):
        (ln,) = struct.unpack_from("<I", foot, off)
        off += 4
        name = foot[off: off + ln].decode()
        off += ln
        schema.append((name, "float64" if foot[off] == 1 else "int64"))
        off += 1
    return schema


def inspect(path):
    """parse_footer_file summary: rows, codec, row_groups, schema [(name, type)]."""
    rows, nc, groups, codec = ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_uint64(), ctypes.c_int()
    _check(lib().psg_psto_inspect(path.encode(), ctypes.byref(rows), ctypes.byref(nc), ctypes.byref(groups),
                                  ctypes.byref(codec)))
    return {"rows": rows.value, "codec": "block" if codec.value == 1 else "identity", "row_groups": groups.value,
            "schema": _footer_schema(path)}


def gen_workload(kind, out_dir, devices=2, nodes=2, scale=0.01, seed=42, codec="block", row_group_bytes=1 << 20,
                 threads=3, build_rows=120_000, probe_rows=320_000, payload_cols=3, hit_ratio=0.5):
    """gen_workload(kind='tpch') (bench.cpp:85-114), byte-identical to the reference generator.

    Defaults mirror the reference's (bindings.cpp:180-193 + GenWorkloadSpec, bench.hpp:51): the zlib
    block codec, whose chunks the GPU inflates in HBM; codec='identity' writes raw column chunks.
    kind='synthetic' writes the synthetic join tables (SyntheticJoinSpec defaults, workload.hpp:27-33);
    any other kind is the TPC-H analog, as in the reference's binding."""
    if kind == "synthetic":  # the reference's pybind maps any other kind to tpch (bindings.cpp:184)
        _check(lib().psg_gen_synthetic(out_dir.encode(), int(nodes), int(devices), int(seed),
                                       1 if codec == "block" else 0, int(row_group_bytes), int(build_rows),
                                       int(probe_rows), int(payload_cols), float(hit_ratio)))
        return os.path.join(out_dir, "manifest.json")
    _check(lib().psg_gen_tpch(out_dir.encode(), float(scale), int(nodes), int(devices), int(seed),
                              1 if codec == "block" else 0, int(row_group_bytes), int(threads)))
    return os.path.join(out_dir, "manifest.json")


def run_plan(plan, data_root, mode="overlapped", ctx: Context | None = None) -> Result:
    """execute_plan on this process's GPU (one rank). Returns this rank's PipelineResult."""
    return (ctx or _ctx()).execute_plan(plan, data_root, mode)


def _atoms(predicate):
    atoms = []
    for col, op, lit in predicate or []:
        a = Atom()
        a.column = col.encode()
        a.op = op.encode()
        a.literal_is_float = 1 if isinstance(lit, float) else 0
        a.literal_i = int(lit) if not isinstance(lit, float) else 0
        a.literal_f = float(lit)
        atoms.append(a)
    arr = (Atom * max(len(atoms), 1))(*atoms)
    return arr, len(atoms)


def filter(columns: dict, predicate, ctx: Context | None = None, types=None) -> Result:
    """Order-preserving filter (ops.cpp:45-54) on the GPU."""
    b = _make_batch(columns, types)
    arr, n = _atoms(predicate)
    out = ctypes.c_void_p()
    _check(lib().psg_filter((ctx or _ctx())._h, ctypes.byref(b), arr, n, ctypes.byref(out)))
    return Result(out)


def partition(columns: dict, key, nparts, hash_kind="multiply_shift", ctx: Context | None = None, types=None):
    """partition (ops.cpp:56-78): returns [Result-like dict per part] preserving order within parts."""
    b = _make_batch(columns, types)
    counts = (ctypes.c_uint64 * nparts)()
    out = ctypes.c_void_p()
    _check(lib().psg_partition((ctx or _ctx())._h, ctypes.byref(b), key.encode(), int(nparts),
                               1 if hash_kind == "identity" else 0, ctypes.byref(out), counts))
    r = Result(out)
    parts, at = [], 0
    for p in range(nparts):
        parts.append(r.rows[at: at + counts[p]])
        at += counts[p]
    return r.schema, parts


class HashTable:
    """HashTable (ops.hpp:49-82) on the GPU: build over several batches of one schema (duplicates
    keep every row), then lookup / probe any number of times. Mirrors the reference's
    HashTable::build(batches, key, hash) / lookup(key) / probe(batch, key) / row_count /
    key_at / payload_at."""

    def __init__(self, handle, ctx, key):
        self._h, self._ctx, self._key = handle, ctx, key
        rows, nc = ctypes.c_uint64(), ctypes.c_uint32()
        _check(lib().psg_hashtable_shape(self._h, ctypes.byref(rows), ctypes.byref(nc)))
        self._rows, self._npay = rows.value, nc.value

    @classmethod
    def build(cls, batches, key_column, hash="multiply_shift", ctx: Context | None = None, types=None):
        ctx = ctx or _ctx()
        bs = [_make_batch(b, types) for b in batches]
        arr = (Batch * max(len(bs), 1))(*bs)
        out = ctypes.c_void_p()
        _check(lib().psg_hashtable_build(ctx._h, arr, len(bs), key_column.encode(),
                                         1 if hash == "identity" else 0, ctypes.byref(out)))
        t = cls(out, ctx, key_column)
        t._keep = bs
        return t

    def row_count(self):
        return self._rows

    def key_at(self, row):
        k = ctypes.c_int64()
        pay = (ctypes.c_uint64 * max(self._npay, 1))()
        _check(lib().psg_hashtable_row(self._h, self._key.encode(), int(row), ctypes.byref(k), pay))
        return k.value

    def payload_at(self, col, row):
        k = ctypes.c_int64()
        pay = (ctypes.c_uint64 * max(self._npay, 1))()
        _check(lib().psg_hashtable_row(self._h, self._key.encode(), int(row), ctypes.byref(k), pay))
        return pay[col]

    def lookup_many(self, keys):
        """[indices of the build rows carrying key] for every key (one GPU pass)."""
        ks = np.ascontiguousarray(np.asarray(keys, dtype=np.int64))
        n = len(ks)
        offs = np.zeros(n + 1, dtype=np.uint64)
        total = ctypes.c_uint64()
        cap = max(n, 1) * 4
        while True:
            rows = np.zeros(cap, dtype=np.uint64)
            rc = lib().psg_hashtable_lookup(self._ctx._h, self._h, ks.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), n,
                                            offs.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                            rows.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), cap,
                                            ctypes.byref(total))
            if rc == 0:
                break
            if total.value > cap:
                cap = int(total.value)
                continue
            _check(rc)
        return [rows[int(offs[i]):int(offs[i + 1])].tolist() for i in range(n)]

    def lookup(self, key):
        return self.lookup_many([key])[0]

    def probe(self, batch: dict, probe_key, types=None) -> "Result":
        pb = _make_batch(batch, types)
        out = ctypes.c_void_p()
        _check(lib().psg_hashtable_probe(self._ctx._h, self._h, ctypes.byref(pb), probe_key.encode(), ctypes.byref(out)))
        return Result(out)

    def free(self):
        if getattr(self, "_h", None):
            lib().psg_hashtable_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def concat(batches, ctx: Context | None = None, types=None) -> "Result":
    """concat (ops.cpp:80-98): batches of one schema into one batch."""
    bs = [_make_batch(b, types) for b in batches]
    arr = (Batch * max(len(bs), 1))(*bs)
    out = ctypes.c_void_p()
    _check(lib().psg_concat((ctx or _ctx())._h, arr, len(bs), ctypes.byref(out)))
    return Result(out)


def hash_join(build: dict, build_key, probe: dict, probe_key, ctx: Context | None = None, build_types=None,
              probe_types=None) -> Result:
    """HashTable::build + probe (ops.cpp:105-222): build payload ++ probe columns, multiset order."""
    bb = _make_batch(build, build_types)
    pb = _make_batch(probe, probe_types)
    out = ctypes.c_void_p()
    _check(lib().psg_hash_join((ctx or _ctx())._h, ctypes.byref(bb), build_key.encode(), ctypes.byref(pb),
                               probe_key.encode(), ctypes.byref(out)))
    return Result(out)


def codec_decompress(chunks, sizes, codec="block", ctx: Context | None = None):
    """codec_decompress (psto.cpp:133-143) for a batch of chunks, inflated on the GPU.

    ``chunks``: bytes-like compressed streams; ``sizes``: their exact uncompressed sizes. Returns
    a list of ``bytes``. Raises PsgError(IoFailure) on any invalid stream, like the reference."""
    n = len(chunks)
    if len(sizes) != n:
        raise ValueError("chunks and sizes differ in length")
    srcs = [bytes(c) for c in chunks]
    outs = [ctypes.create_string_buffer(max(int(z), 1)) for z in sizes]
    src_p = (ctypes.c_void_p * max(n, 1))(*[ctypes.cast(ctypes.c_char_p(b), ctypes.c_void_p) for b in srcs])
    dst_p = (ctypes.c_void_p * max(n, 1))(*[ctypes.cast(o, ctypes.c_void_p) for o in outs])
    src_l = (ctypes.c_uint64 * max(n, 1))(*[len(b) for b in srcs])
    dst_l = (ctypes.c_uint64 * max(n, 1))(*[int(z) for z in sizes])
    kind = {"identity": 0, "block": 1}[codec] if isinstance(codec, str) else int(codec)
    _check(lib().psg_codec_decompress((ctx or _ctx())._h, kind, n, src_p, src_l, dst_p, dst_l))
    return [o.raw[:int(z)] for o, z in zip(outs, sizes)]


def scan(path, predicate=None, ctx: Context | None = None):
    """Reads a PSTO table through the GPU filter (read_blocking + filter, scan.cpp:273-336)."""
    meta = inspect(path)
    import struct
    with open(path, "rb") as f:
        data = f.read()
    # footer walk for chunk offsets
    (flen,) = struct.unpack_from("<Q", data, len(data) - 12)
    foot = data[len(data) - 12 - flen: len(data) - 12]
    off = 5
    (nc,) = struct.unpack_from("<I", foot, off)
    off += 4
    for _ in range(nc):
        (ln,) = struct.unpack_from("<I", foot, off)
        off += 4 + ln + 1
    (ng,) = struct.unpack_from("<I", foot, off)
    off += 4
    cols = [[] for _ in range(nc)]
    pending = []  # block codec: (col, stream, usize), inflated on the GPU in one batch
    for _ in range(ng):
        (rows,) = struct.unpack_from("<Q", foot, off)
        off += 8
        for c in range(nc):
            o, cs, us, _mn, _mx = struct.unpack_from("<5Q", foot, off)
            off += 40
            if meta["codec"] == "identity":
                cols[c].append(np.frombuffer(data, dtype="<u8", count=rows, offset=o))
            else:
                pending.append((c, data[o:o + cs], us))
    if pending:
        raw = codec_decompress([p[1] for p in pending], [p[2] for p in pending], "block", ctx=ctx)
        for (c, _s, _u), r in zip(pending, raw):
            cols[c].append(np.frombuffer(r, dtype="<u8"))
    schema = meta["schema"]
    columns = {n: (np.concatenate(cols[i]) if cols[i] else np.zeros(0, np.uint64)) for i, (n, _t) in enumerate(schema)}
    types = {n: (1 if t == "float64" else 0) for n, t in schema}
    res = filter(columns, predicate or [], ctx=ctx, types=types)
    return res.to_dict()
