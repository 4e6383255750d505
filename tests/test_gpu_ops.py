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
