"""GPU inflate of the PSTO block codec (zlib streams) against zlib itself and the reference.

codec_decompress (psto.cpp:133-143) calls zlib's uncompress and raises IoFailure("inflate
failed") unless the stream decodes to exactly the expected size; psg_codec_decompress runs the
same contract on the GPU kernel the scan path uses (inflate.cu). Streams cover every deflate
block type (stored, fixed, dynamic) through zlib levels and strategies; corrupted streams must
fail exactly when zlib's uncompress would. The end-to-end cases run execute_plan over block-coded
tables and compare with the reference's golden results / the oracle.
"""
import json
import zlib

import numpy as np
import pytest

import paper_2512_02862_b200 as psg
from oracle import plan_oracle as po

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = psg.Context(0)
    c.set_ingest(io_threads=4, batch_bytes=4 << 20)
    yield c
    c.close()


def _payloads(rng):
    """Byte strings shaped like PSTO column chunks and a few adversarial ones."""
    out = []
    n = 32768
    out.append(rng.integers(0, 6_000_000, n).astype("<i8").tobytes())            # orderkey-like
    out.append(np.sort(rng.integers(0, 1 << 40, n)).astype("<i8").tobytes())      # sorted wide ints
    out.append(rng.integers(0, 11, n).astype("<i8").tobytes())                    # discount-like
    out.append(rng.normal(size=n).astype("<f8").tobytes())                        # doubles
    out.append(np.repeat(rng.integers(0, 1 << 30, n // 64), 64).astype("<i8").tobytes())  # long runs
    out.append(rng.integers(0, 256, 100_003, dtype=np.uint8).tobytes())           # incompressible
    out.append(b"\x00" * 70_001)                                                  # dist-1 runs
    out.append(b"")                                                               # empty
    out.append(b"x")
    out.append(bytes(range(256)) * 37 + b"tail")                                   # short periods
    return out


def _uncompress_ok(stream, usize):
    """zlib's uncompress(dest_len=usize) success, as codec_decompress sees it."""
    d = zlib.decompressobj()
    try:
        out = d.decompress(stream, usize + 1)
    except zlib.error:
        return False, None
    return d.eof and len(out) == usize, out


def test_inflate_matches_zlib_all_block_types(ctx):
    rng = np.random.default_rng(7)
    chunks, sizes, want = [], [], []
    for data in _payloads(rng):
        for level in (0, 1, 6, 9):
            chunks.append(zlib.compress(data, level))
            sizes.append(len(data))
            want.append(data)
        for strategy in (zlib.Z_FIXED, zlib.Z_HUFFMAN_ONLY, zlib.Z_RLE, zlib.Z_FILTERED):
            c = zlib.compressobj(6, zlib.DEFLATED, 15, 8, strategy)
            chunks.append(c.compress(data) + c.flush())
            sizes.append(len(data))
            want.append(data)
        # sync-flushed stream: empty stored blocks between data blocks
        c = zlib.compressobj(1)
        half = len(data) // 2
        chunks.append(c.compress(data[:half]) + c.flush(zlib.Z_SYNC_FLUSH) + c.compress(data[half:]) + c.flush())
        sizes.append(len(data))
        want.append(data)
    got = psg.codec_decompress(chunks, sizes, "block", ctx=ctx)
    for i, (g, w) in enumerate(zip(got, want)):
        assert g == w, i


def test_inflate_psto_chunks_one_batch(ctx, tmp_path):
    """Every chunk of a block-coded PSTO file, inflated in one launch, equals the identity file."""
    psg.gen_workload("tpch", str(tmp_path / "b"), devices=1, nodes=1, scale=0.02, seed=3, codec="block")
    psg.gen_workload("tpch", str(tmp_path / "i"), devices=1, nodes=1, scale=0.02, seed=3, codec="identity")
    for t in ("lineitem.node0", "orders.node0", "customer"):
        b = psg.scan(str(tmp_path / "b" / "dev0" / (t + ".psto")), ctx=ctx)
        i = psg.scan(str(tmp_path / "i" / "dev0" / (t + ".psto")), ctx=ctx)
        assert b.keys() == i.keys()
        for k in b:
            assert np.array_equal(np.asarray(b[k]), np.asarray(i[k])), (t, k)


def test_inflate_errors_like_uncompress(ctx):
    rng = np.random.default_rng(11)
    data = rng.integers(0, 1000, 4096).astype("<i8").tobytes()
    good = zlib.compress(data, 1)
    cases = []
    cases.append((good, len(data) - 1))          # stream longer than the buffer
    cases.append((good, len(data) + 1))          # short output
    cases.append((good[:-5], len(data)))         # truncated
    cases.append((b"\x78\x9c" + b"\xff" * 40, 100))  # reserved block type
    cases.append((b"\x79\x9c" + good[2:], len(data)))  # bad header check
    bad_adler = bytearray(good)
    bad_adler[-1] ^= 1
    cases.append((bytes(bad_adler), len(data)))
    cases.append((b"", 0))
    for stream, usize in cases:
        ok, _ = _uncompress_ok(stream, usize)
        assert not ok
        with pytest.raises(psg.PsgError) as e:
            psg.codec_decompress([stream], [usize], "block", ctx=ctx)
        assert e.value.kind == "IoFailure" and "inflate failed" in str(e.value)
    # random bit flips: fail exactly when zlib fails, else produce zlib's bytes
    for trial in range(200):
        b = bytearray(good)
        pos = int(rng.integers(0, len(b)))
        b[pos] ^= 1 << int(rng.integers(0, 8))
        ok, out = _uncompress_ok(bytes(b), len(data))
        if ok:
            assert psg.codec_decompress([bytes(b)], [len(data)], "block", ctx=ctx)[0] == out
        else:
            with pytest.raises(psg.PsgError):
                psg.codec_decompress([bytes(b)], [len(data)], "block", ctx=ctx)
    # one bad stream fails the whole batch (the reference throws on the first bad chunk)
    with pytest.raises(psg.PsgError):
        psg.codec_decompress([good, good[:-5]], [len(data)] * 2, "block", ctx=ctx)


@pytest.fixture(scope="module")
def bdata(tmp_path_factory):
    base = tmp_path_factory.mktemp("bdata")
    cache = {}

    def get(scale, seed=42, rg=1 << 20, codec="block"):
        key = (scale, seed, rg, codec)
        if key not in cache:
            d = str(base / ("d%d" % len(cache)))
            psg.gen_workload("tpch", d, devices=1, nodes=1, scale=scale, seed=seed, row_group_bytes=rg, codec=codec)
            cache[key] = d
        return cache[key]

    return get


@pytest.mark.parametrize("mode", ["overlapped", "blocking", "fastio", "combined"])
def test_block_codec_golden(ctx, bdata, golden, mode):
    """The reference's block-codec acceptance case (results.json) on GPU-inflated chunks."""
    cases = [r for r in golden["results"] if r["codec"] == "block"]
    assert cases
    for r in cases:
        d = bdata(r["scale"], r["seed"], r["rg_bytes"])
        s = po.summary([(lambda x: (x.schema, x.rows))(ctx.execute_plan(golden["plans"][r["plan"]], d, mode))])
        assert (s["rows"], s["rowhash"], s["colsums"]) == (r["rows"], r["rowhash"], r["colsums"]), (r["case"], mode)


def test_block_codec_plans_vs_identity(ctx, bdata, golden):
    """Every golden plan gives identical rows over block-coded and identity-coded copies of the
    same tables (streaming, staged and small-batch paths)."""
    for pname in ("canonical", "projection_buildsums", "multi_atom", "global_agg", "no_aggregate", "float_literal",
                  "empty"):
        plan = golden["plans"][pname]
        ident = ctx.execute_plan(plan, bdata(0.05, codec="identity"), "overlapped")
        blk = ctx.execute_plan(plan, bdata(0.05), "overlapped")
        want = po.summary([(ident.schema, ident.rows)])
        assert blk.schema == ident.schema and po.summary([(blk.schema, blk.rows)]) == want, pname
        st = ctx.stage_plan(plan, bdata(0.05))
        r = st.run()
        assert po.summary([(r.schema, r.rows)]) == want, pname
        st.free()


def test_block_codec_sf1_golden(ctx, bdata, golden):
    r = [x for x in golden["results"] if x["plan"] == "canonical" and x["scale"] == 1.0][0]
    res = ctx.execute_plan(golden["plans"]["canonical"], bdata(1.0), "overlapped")
    s = po.summary([(res.schema, res.rows)])
    assert (s["rows"], s["rowhash"], s["colsums"]) == (r["rows"], r["rowhash"], r["colsums"])
    assert res.stats["ingest_bytes"] > 0


def test_block_codec_corrupt_chunk_raises(ctx, bdata, golden, tmp_path):
    """A flipped byte inside a compressed chunk -> IoFailure("inflate failed"), like decode_group."""
    import shutil
    d = str(tmp_path / "c")
    shutil.copytree(bdata(0.01), d)
    f = d + "/dev0/lineitem.node0.psto"
    raw = bytearray(open(f, "rb").read())
    raw[200] ^= 0xFF
    open(f, "wb").write(bytes(raw))
    for mode in ("overlapped", "blocking"):
        with pytest.raises(psg.PsgError) as e:
            ctx.execute_plan(golden["plans"]["canonical"], d, mode)
        assert e.value.kind == "IoFailure"
