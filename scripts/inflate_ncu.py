"""Measurement tool: one k_inflate launch over the lineitem chunks of a block-coded SF1 table
(ncu target; not product code).  python scripts/inflate_ncu.py [--jobs N]"""
import argparse
import os
import struct
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_02862_b200 as psg  # noqa: E402


def chunks_of(path):
    data = open(path, "rb").read()
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
    out = []
    for _ in range(ng):
        off += 8
        for _c in range(nc):
            o, cs, us, _mn, _mx = struct.unpack_from("<5Q", foot, off)
            off += 40
            out.append((data[o:o + cs], us))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=592)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--scale", type=float, default=1.0)
    a = ap.parse_args()
    d = "/tmp/psg_inflate/sf%g_block" % a.scale
    if not os.path.exists(d + "/DONE"):
        psg.gen_workload("tpch", d, devices=1, nodes=1, scale=a.scale, seed=42, codec="block")
        open(d + "/DONE", "w").write("ok")
    ch = chunks_of(d + "/dev0/lineitem.node0.psto")[:a.jobs]
    ctx = psg.Context(0)
    for _ in range(a.reps):
        t = time.time()
        out = psg.codec_decompress([c for c, _ in ch], [u for _, u in ch], "block", ctx=ctx)
        dt = time.time() - t
        print("%d chunks, %.1f MB decoded in %.1f ms (host API incl. copies)" % (
            len(ch), sum(len(x) for x in out) / 1e6, dt * 1e3), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
