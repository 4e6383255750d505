"""ORACLE — test infrastructure only (never imported by the product path).

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference``
leg may import this module, and only as the checker / CPU baseline, never as the thing measured.

numpy restatement of the reference plan executor's *result semantics* for the distributed
storage-resident OLAP path (``execute_plan``):

* plan parsing ............ /root/reference/proj/src/pipeline.cpp:108-156 (``{data}``/``{node}``/
                            ``{nodes}`` substitution, one-component ``*`` glob :57-84),
                            validation :178-196
* PSTO footer/reader ...... /root/reference/proj/src/psto.cpp:231-292 (footer), :133-142 (codecs)
* projection .............. /root/reference/proj/src/scan.cpp:121-137
* filter / predicate ...... /root/reference/proj/src/ops.cpp:45-54, predicate.cpp:43-110
                            (literal cast ``literal_as<T>`` :69-74)
* local join chain ........ pipeline.cpp:431-448 -> HashTable::probe ops.cpp:173-222
                            (output = build payload ++ probe columns, ``_p`` on name clash)
* shuffle ................. partition_of = ((k*0x9E3779B97F4A7C15) >> 13) % n, hashing.hpp:26-37
* aggregate ............... HashAggregator pipeline.cpp:256-305 (count, wrapping int64 sums,
                            double sums; grouped rows in signed key order; a global aggregate is
                            one unmerged row per node; empty input -> no row)

Results are per node, exactly like ``PipelineResult.rows`` of every node of a run. The oracle is
pinned against the reference itself (tests/golden/*.json, made by tests/golden/make_golden.py
from oracle/_ref/ref_driver) and against SURVEY.md §8(c)'s golden table.
"""
from __future__ import annotations

import glob as _glob
import json
import os
import struct
import zlib
from dataclasses import dataclass, field

import numpy as np

MULT = np.uint64(0x9E3779B97F4A7C15)
INT64, FLOAT64 = 0, 1


# ----------------------------------------------------------------------------- PSTO reader
@dataclass
class TableMeta:
    names: list
    types: list
    codec: int
    groups: list  # [(rows, [(offset, csize, usize, min_raw, max_raw)] * ncols)]


def parse_footer(path: str) -> TableMeta:
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < 20 or data[:4] != b"PSTO" or data[-4:] != b"PSTO":
        raise ValueError("corrupt footer: bad magic")
    (flen,) = struct.unpack_from("<Q", data, len(data) - 12)
    foot = memoryview(data)[len(data) - 12 - flen: len(data) - 12]
    off = 0

    def take(fmt):
        nonlocal off
        v = struct.unpack_from(fmt, foot, off)
        off += struct.calcsize(fmt)
        return v

    (ver,) = take("<I")
    if ver != 1:
        raise ValueError("corrupt footer: version")
    (codec,) = take("<B")
    (ncols,) = take("<I")
    names, types = [], []
    for _ in range(ncols):
        (ln,) = take("<I")
        names.append(bytes(foot[off: off + ln]).decode())
        off += ln
        (t,) = take("<B")
        types.append(t)
    (ngroups,) = take("<I")
    groups = []
    for _ in range(ngroups):
        (rows,) = take("<Q")
        cols = [take("<5Q") for _ in range(ncols)]
        groups.append((rows, cols))
    return TableMeta(names, types, codec, groups)


def read_table(path: str, meta: TableMeta | None = None) -> dict:
    """Whole-file read: {name: np.ndarray(uint64 raw words)} in file column order."""
    meta = meta or parse_footer(path)
    with open(path, "rb") as f:
        data = f.read()
    out = {n: [] for n in meta.names}
    for rows, cols in meta.groups:
        for n, (offset, csize, usize, _mn, _mx) in zip(meta.names, cols):
            raw = data[offset: offset + csize]
            if meta.codec == 1:
                raw = zlib.decompress(raw)
            out[n].append(np.frombuffer(raw, dtype="<u8", count=rows))
    return {n: (np.concatenate(v) if v else np.zeros(0, np.uint64)) for n, v in out.items()}


# ----------------------------------------------------------------------------- plan
def _substitute(s, data_root, node, nodes):
    return s.replace("{data}", data_root).replace("{node}", str(node)).replace("{nodes}", str(nodes))


def expand_glob(pattern: str) -> list:
    if "*" not in pattern:
        return [pattern] if os.path.exists(pattern) else []
    return sorted(_glob.glob(pattern))


@dataclass
class Scan:
    table: str
    paths: list
    columns: list
    predicate: list  # [(col, op, literal)] ; literal int or float
    replicated: bool = False


@dataclass
class Join:
    id: str
    build: str
    probe: str
    build_key: str
    probe_key: str
    shuffle: bool


@dataclass
class Plan:
    scans: list
    joins: list
    aggregate: dict | None
    raw: dict = field(default_factory=dict)


def parse_plan(text: str, data_root: str, node: int, nodes: int, local: bool = False) -> Plan:
    """local=True: the no-shuffle plans of psg_execute_local (exactly zero shuffled joins)."""
    j = json.loads(text)
    scans = []
    for s in j["scans"]:
        paths = []
        for p in s["paths"]:
            exp = expand_glob(_substitute(p, data_root, node, nodes))
            if not exp:
                raise FileNotFoundError("io failure: no files match scan path: " + p)
            paths += exp
        pred = [(a["col"], a["op"], a["value"]) for a in s.get("predicate", [])]
        scans.append(Scan(s["table"], paths, list(s.get("columns", [])), pred, bool(s.get("replicated", False))))
    joins = [Join(x["id"], x["build"], x["probe"], x["build_key"], x["probe_key"], x.get("mode", "replicated") == "shuffle")
             for x in j.get("joins", [])]
    agg = None
    if "aggregate" in j:
        agg = {"group_by": j["aggregate"].get("group_by", ""), "sums": list(j["aggregate"].get("sums", []))}
    plan = Plan(scans, joins, agg, j)
    shuffles = [x for x in joins if x.shuffle]
    if local:
        if shuffles or not agg or agg["group_by"]:
            raise ValueError("invalid input: local plans have no shuffled join and end in a global aggregate")
        return plan
    if len(shuffles) != 1:
        raise ValueError("invalid input: plans currently require one shuffled join")
    if agg and agg["group_by"] and agg["group_by"] != shuffles[0].probe_key:
        raise ValueError("invalid input: group key must match the shuffle probe key so groups co-locate")
    return plan


# ----------------------------------------------------------------------------- operators
class Batch:
    """Columnar batch of raw uint64 words with a schema [(name, type)]."""

    def __init__(self, fields, cols):
        self.fields = list(fields)
        self.cols = list(cols)

    @property
    def rows(self):
        return 0 if not self.cols else len(self.cols[0])

    def idx(self, name):
        for i, (n, _t) in enumerate(self.fields):
            if n == name:
                return i
        raise KeyError("unknown column: " + name)

    def take(self, sel):
        return Batch(self.fields, [c[sel] for c in self.cols])


def _cmp(a, op, b):
    return {"<": a < b, "<=": a <= b, "==": a == b, "=": a == b, "!=": a != b, ">=": a >= b, ">": a > b}[op]


def filter_mask(b: Batch, pred) -> np.ndarray:
    m = np.ones(b.rows, dtype=bool)
    for col, op, lit in pred:
        i = b.idx(col)
        t = b.fields[i][1]
        if t == INT64:
            v = b.cols[i].view(np.int64)
            litv = np.int64(int(lit))  # static_cast<int64_t>(double) truncates toward zero
        else:
            v = b.cols[i].view(np.float64)
            litv = np.float64(lit)
        m &= _cmp(v, op, litv)
    return m


def scan_table(scan: Scan, path: str) -> Batch:
    meta = parse_footer(path)
    cols = read_table(path, meta)
    if scan.columns:
        for c in scan.columns:
            if c not in meta.names:
                raise KeyError("unknown column: " + c)
        names = [n for n in meta.names if n in scan.columns]
    else:
        names = list(meta.names)
    fields = [(n, meta.types[meta.names.index(n)]) for n in names]
    b = Batch(fields, [cols[n] for n in names])
    return b.take(filter_mask(b, scan.predicate))


def concat(batches):
    batches = [b for b in batches if b is not None]
    if not batches:
        return None
    return Batch(batches[0].fields, [np.concatenate([b.cols[i] for b in batches]) for i in range(len(batches[0].fields))])


def hash_join(build: Batch, build_key: str, probe: Batch, probe_key: str) -> Batch:
    """Inner join: output = build payload (all but the key) ++ probe columns (``_p`` on clash)."""
    bk = build.cols[build.idx(build_key)].view(np.int64)
    pk = probe.cols[probe.idx(probe_key)].view(np.int64)
    order = np.argsort(bk, kind="stable")
    sk = bk[order]
    lo = np.searchsorted(sk, pk, "left")
    hi = np.searchsorted(sk, pk, "right")
    cnt = hi - lo
    total = int(cnt.sum())
    pidx = np.repeat(np.arange(len(pk)), cnt)
    starts = np.repeat(lo, cnt)
    within = np.arange(total) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    bidx = order[starts + within]
    fields, cols = [], []
    kidx = build.idx(build_key)
    for i, f in enumerate(build.fields):
        if i == kidx:
            continue
        fields.append(f)
        cols.append(build.cols[i][bidx])
    names = {f[0] for f in fields}
    for i, (n, t) in enumerate(probe.fields):
        fields.append((n + "_p" if n in names else n, t))
        cols.append(probe.cols[i][pidx])
    return Batch(fields, cols)


def partition_of(keys_raw: np.ndarray, n: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        h = (keys_raw.astype(np.uint64) * MULT) >> np.uint64(13)
    return (h % np.uint64(n)).astype(np.int64)


def aggregate(b: Batch, group_by: str, sums: list):
    """HashAggregator restated. Returns (schema, rows[list of tuples of uint64 words])."""
    sum_idx = [b.idx(c) for c in sums]
    schema = ([b.fields[b.idx(group_by)]] if group_by else []) + [("rows", INT64)] + \
        [("sum_" + b.fields[i][0], b.fields[i][1]) for i in sum_idx]
    if b.rows == 0:
        return schema, np.zeros((0, len(schema)), np.uint64)
    if group_by:
        keys = b.cols[b.idx(group_by)].view(np.int64)
        uk, inv = np.unique(keys, return_inverse=True)
    else:
        uk, inv = np.zeros(1, np.int64), np.zeros(b.rows, np.int64)
    order = np.argsort(inv, kind="stable")
    sinv = inv[order]
    starts = np.flatnonzero(np.r_[True, sinv[1:] != sinv[:-1]])
    out = []
    if group_by:
        out.append(uk.view(np.uint64))
    out.append(np.bincount(inv, minlength=len(uk)).astype(np.uint64))
    for i in sum_idx:
        col = b.cols[i][order]
        if b.fields[i][1] == INT64:
            with np.errstate(over="ignore"):
                s = np.add.reduceat(col.astype(np.uint64), starts)  # wraps mod 2^64
            out.append(s.astype(np.uint64))
        else:
            out.append(np.add.reduceat(col.view(np.float64), starts).view(np.uint64))
    return schema, np.stack(out, axis=1)


# ----------------------------------------------------------------------------- executor
def _source(plan: Plan, name: str):
    for s in plan.scans:
        if s.table == name:
            return s, []
    for j in plan.joins:
        if j.id == name:
            base, chain = _source(plan, j.probe)
            return base, chain + [j]
    raise ValueError("plan references unknown stream: " + name)


def _local_tables(plan: Plan):
    tables = {}
    for j in plan.joins:
        if j.shuffle:
            continue
        s = next(x for x in plan.scans if x.table == j.build)
        if not s.replicated:
            raise ValueError("invalid input: local join must build from a replicated scan")
        tables[j.id] = concat([scan_table(s, p) for p in s.paths])
    return tables


def _stream(plan: Plan, name: str, tables):
    base, chain = _source(plan, name)
    b = concat([scan_table(base, p) for p in base.paths])
    if b is None:
        return None
    for j in chain:
        b = hash_join(tables[j.id], j.build_key, b, j.probe_key)
    return b


def execute(plan_text: str, data_root: str, nodes: int):
    """Returns [(schema, rows ndarray[uint64] (nrows, ncols))] per node."""
    plans = [parse_plan(plan_text, data_root, k, nodes) for k in range(nodes)]
    shuffle = next(j for j in plans[0].joins if j.shuffle)
    builds, probes = [], []
    for k in range(nodes):
        tables = _local_tables(plans[k])
        builds.append(_stream(plans[k], shuffle.build, tables))
        probes.append(_stream(plans[k], shuffle.probe, tables))
    build_all = concat(builds)
    probe_all = concat(probes)
    results = []
    if build_all is None or probe_all is None:
        return [([], np.zeros((0, 0), np.uint64)) for _ in range(nodes)]
    bpart = partition_of(build_all.cols[build_all.idx(shuffle.build_key)], nodes)
    ppart = partition_of(probe_all.cols[probe_all.idx(shuffle.probe_key)], nodes)
    agg = plans[0].aggregate
    for k in range(nodes):
        joined = hash_join(build_all.take(bpart == k), shuffle.build_key, probe_all.take(ppart == k), shuffle.probe_key)
        if agg is not None:
            results.append(aggregate(joined, agg["group_by"], agg["sums"]))
        else:
            rows = np.stack(joined.cols, axis=1) if joined.cols else np.zeros((0, 0), np.uint64)
            results.append((joined.fields, rows))
    return results


def execute_local(plan_text: str, data_root: str, nodes: int):
    """Local plans (no shuffled join; the psg_execute_local extension): per node, the root stream
    (scan or replicated-join chain, _stream above) reduced to one global-aggregate partial row,
    the semantics of execute_plan's global aggregate (pipeline.cpp:277-281, 892-897).
    Returns [(schema, rows)] per node."""
    results = []
    for k in range(nodes):
        plan = parse_plan(plan_text, data_root, k, nodes, local=True)
        consumed = {j.build for j in plan.joins} | {j.probe for j in plan.joins}
        roots = [j.id for j in plan.joins if j.id not in consumed] + \
                [s.table for s in plan.scans if not s.replicated and s.table not in consumed]
        assert len(roots) == 1, roots
        tables = _local_tables(plan)
        stream = _stream(plan, roots[0], tables)
        results.append(aggregate(stream, "", plan.aggregate["sums"]) if stream is not None
                       else ([], np.zeros((0, 0), np.uint64)))
    return results


def fnv1a64_rows(rows: np.ndarray) -> int:
    """sum over rows of FNV-1a64 of the row's little-endian words (mod 2^64), vectorised."""
    if rows.size == 0:
        return 0
    b = np.ascontiguousarray(rows.astype("<u8")).view(np.uint8).reshape(rows.shape[0], -1)
    h = np.full(rows.shape[0], 0xCBF29CE484222325, dtype=np.uint64)
    p = np.uint64(0x100000001B3)
    with np.errstate(over="ignore"):
        for i in range(b.shape[1]):
            h ^= b[:, i].astype(np.uint64)
            h *= p
        return int(h.sum(dtype=np.uint64))


def summary(per_node) -> dict:
    rows = [r for _s, r in per_node if r.size]
    allr = np.concatenate(rows) if rows else np.zeros((0, 0), np.uint64)
    with np.errstate(over="ignore"):
        colsums = [str(int(x)) for x in allr.sum(axis=0, dtype=np.uint64)] if allr.size else []
    return {"rows": int(allr.shape[0]), "rowhash": "%016x" % fnv1a64_rows(allr), "colsums": colsums,
            "per_node_rows": [int(r.shape[0]) for _s, r in per_node]}
