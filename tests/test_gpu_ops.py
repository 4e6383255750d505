"""Operator-level parity (ops.hpp:35-83) on the GPU, after core_ops_test.cpp's cases."""
import numpy as np
import pytest

import paper_2512_02862_b200 as psg
from oracle import plan_oracle as po

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = psg.Context(0)
    yield c
    c.close()


def test_filter_keeps_qualifying_rows_in_order(ctx):
    r = psg.filter({"k": [1, 2, 3]}, [("k", "<", 3)], ctx=ctx)
    assert r.column("k").tolist() == [1, 2]


def test_filter_empty_and_unknown_column(ctx):
    r = psg.filter({"k": np.zeros(0, np.int64)}, [("k", ">", 0)], ctx=ctx)
    assert r.rows.shape == (0, 1)
    with pytest.raises(psg.PsgError) as e:
        psg.filter({"k": [1]}, [("zzz", "<", 1)], ctx=ctx)
    assert e.value.kind == "UnknownColumn"


@pytest.mark.parametrize("n", [10_000, 1_000_003])
def test_filter_matches_scalar_oracle_multi_atom_float(ctx, n):
    rng = np.random.default_rng(20250810)
    k = rng.integers(0, 1_000_000, n)
    v = rng.random(n)
    w = rng.integers(-5, 5, n)
    pred = [("k", "<", 300_000), ("v", ">=", 0.25), ("w", "!=", 0)]
    got = psg.filter({"k": k, "v": v, "w": w}, pred, ctx=ctx)
    m = (k < 300_000) & (v >= 0.25) & (w != 0)
    assert np.array_equal(got.column("k"), k[m])
    assert np.array_equal(got.column("v"), v[m])
    assert np.array_equal(got.column("w"), w[m])


def test_partition_identity_hash(ctx):
    schema, parts = psg.partition({"k": [3, 4, 7, 10]}, "k", 2, "identity", ctx=ctx)
    assert parts[0][:, 0].tolist() == [4, 10]
    assert parts[1][:, 0].tolist() == [3, 7]


def test_partition_50k_matches_reference_order(ctx):
    rng = np.random.default_rng(7)
    keys = rng.integers(-1_000_000, 1_000_000, 50_000)
    vals = np.arange(50_000)
    schema, parts = psg.partition({"k": keys, "v": vals}, "k", 4, ctx=ctx)
    dest = po.partition_of(keys.view(np.uint64), 4)
    for p in range(4):
        assert np.array_equal(parts[p][:, 0].view(np.int64), keys[dest == p])  # order preserved
        assert np.array_equal(parts[p][:, 1].view(np.int64), vals[dest == p])


def test_partition_one_node_is_identity(ctx):
    _s, parts = psg.partition({"k": [5, 6, 7]}, "k", 1, ctx=ctx)
    assert parts[0][:, 0].tolist() == [5, 6, 7]


def test_probe_emits_payload_then_probe_columns(ctx):
    r = psg.hash_join({"k": [1, 2], "v": [100, 200]}, "k", {"pk": [2, 2, 3]}, "pk", ctx=ctx)
    assert [n for n, _ in r.schema] == ["v", "pk"]
    assert sorted(r.column("v").tolist()) == [200, 200]
    r = psg.hash_join({"k": [1, 2], "v": [100, 200]}, "k", {"pk": [777]}, "pk", ctx=ctx)
    assert r.rows.shape[0] == 0


def test_probe_name_clash_gets_p_suffix(ctx):
    r = psg.hash_join({"k": [1], "x": [5]}, "k", {"k": [1], "x": [9]}, "k", ctx=ctx)
    assert [n for n, _ in r.schema] == ["x", "k", "x_p"]
    assert r.rows.tolist() == [[5, 1, 9]]


def test_probe_with_duplicates_matches_nested_loop(ctx):
    rng = np.random.default_rng(1234)
    bk = rng.integers(0, 200, 500)
    bv = 1000 + np.arange(500)
    pk = rng.integers(0, 300, 800)
    got = psg.hash_join({"k": bk, "v": bv}, "k", {"pk": pk}, "pk", ctx=ctx)
    want = sorted((int(bv[i]), int(p)) for p in pk for i in np.flatnonzero(bk == p))
    assert sorted(map(tuple, got.rows.view(np.int64).tolist())) == want


def test_hash_join_sentinel_key(ctx):
    mn = np.iinfo(np.int64).min
    r = psg.hash_join({"k": [mn, mn, 3], "v": [1, 2, 3]}, "k", {"pk": [mn, 3, 4]}, "pk", ctx=ctx)
    assert sorted(map(tuple, r.rows.view(np.int64).tolist())) == [(1, mn), (2, mn), (3, 3)]


# ---- HashTable handle + concat (ops.hpp:35-82; core_ops_test.cpp:123-202) ----
def test_hashtable_lookup_payload_and_duplicates():
    t = psg.HashTable.build([{"k": [1, 2, 3], "v": [10, 20, 30]}], "k")
    rows = t.lookup(2)
    assert len(rows) == 1 and t.payload_at(0, rows[0]) == 20 and t.key_at(rows[0]) == 2
    dup = psg.HashTable.build([{"k": [5, 5, 6], "v": [1, 2, 3]}], "k")
    assert sorted(dup.payload_at(0, r) for r in dup.lookup(5)) == [1, 2]
    assert dup.lookup(7) == [] and dup.row_count() == 3


def test_hashtable_matches_dict_oracle_on_20k_random_rows():
    rng = np.random.default_rng(17)
    k = rng.integers(0, 5000, 20000)
    v = rng.integers(-1 << 40, 1 << 40, 20000)
    # two build batches: row r of the materialised build side = r-th row of the concatenation
    t = psg.HashTable.build([{"k": k[:7000], "v": v[:7000]}, {"k": k[7000:], "v": v[7000:]}], "k")
    assert t.row_count() == 20000
    oracle = {}
    for r, key in enumerate(k.tolist()):
        oracle.setdefault(key, []).append(r)
    probes = rng.integers(-10, 5100, 3000).tolist()
    got = t.lookup_many(probes)
    for key, rows in zip(probes, got):
        assert sorted(rows) == oracle.get(key, []), key
    assert all(t.key_at(r) == k[r] for r in range(0, 20000, 997))


def test_hashtable_probe_payload_then_probe_columns():
    t = psg.HashTable.build([{"k": [1, 2, 2], "v": [100, 200, 300]}], "k")
    res = t.probe({"pk": [2, 9], "x": [7, 8]}, "pk")
    assert [n for n, _ in res.schema] == ["v", "pk", "x"]
    assert sorted(map(tuple, res.rows.tolist())) == [(200, 2, 7), (300, 2, 7)]
    assert t.probe({"pk": np.zeros(0, np.int64)}, "pk").rows.shape[0] == 0
    assert t.probe({"pk": [42]}, "pk").rows.shape[0] == 0
    clash = t.probe({"v": [5], "k2": [1]}, "k2")
    assert [n for n, _ in clash.schema] == ["v", "v_p", "k2"]


def test_hashtable_probe_agrees_with_nested_loop_oracle():
    rng = np.random.default_rng(3)
    bk, bv, bw = rng.integers(0, 300, 2000), rng.integers(0, 1 << 30, 2000), rng.normal(size=2000)
    pk, px = rng.integers(0, 400, 3000), rng.integers(0, 99, 3000)
    t = psg.HashTable.build([{"k": bk, "v": bv, "w": bw}], "k")
    res = t.probe({"pk": pk, "x": px}, "pk")
    want = []
    by = {}
    for i in range(len(bk)):
        by.setdefault(int(bk[i]), []).append(i)
    for j in range(len(pk)):
        for i in by.get(int(pk[j]), []):
            want.append((int(bv[i]), int(np.float64(bw[i]).view(np.uint64)), int(pk[j]), int(px[j])))
    assert sorted(map(tuple, res.rows.tolist())) == sorted(want)


def test_concat_and_schema_mismatch():
    res = psg.concat([{"a": [1, 2], "b": [3.5, 4.5]}, {"a": [9], "b": [0.25]}])
    assert res.rows[:, 0].tolist() == [1, 2, 9]
    assert res.rows[:, 1].view(np.float64).tolist() == [3.5, 4.5, 0.25]
    with pytest.raises(psg.PsgError) as e:
        psg.concat([{"a": [1]}, {"b": [1]}])
    assert e.value.kind == "InvalidInput"
    with pytest.raises(psg.PsgError):
        psg.HashTable.build([{"k": [1]}, {"k": [2.5]}], "k")
