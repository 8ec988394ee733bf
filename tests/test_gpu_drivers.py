"""Reporting drivers (drivers.py: cmd_sweep / cmd_bench of tools/gradpack_main.cpp)
on the device vs the same loop over the reference's own sources (oracle/_ref):
every sweep container is byte-identical, so relative volume and reconstruction
error agree; the method bench produces a row per CLI method."""
import numpy as np
import pytest
import torch

from oracle.bindings import GpConfig, reference

pytestmark = pytest.mark.gpu


def test_sweep_matches_reference_loop():
    from paper_2102_03112_b200 import Codec
    from paper_2102_03112_b200.dp import hash64, ratio_r
    from paper_2102_03112_b200.drivers import random_r, sweep
    from paper_2102_03112_b200.inputs import normal_f32
    ref = reference()
    if ref is None:
        pytest.skip("oracle/_ref missing")
    dim, ratio, seeds, seed = 5_000, 0.02, 2, 7
    grid = (0.1, 0.01)
    codec = Codec(max_d=dim)
    got = sweep(dim, ratio, seeds, seed, codec=codec, grid=grid).strip().splitlines()[1:]
    codec.close()
    r = ratio_r(dim, ratio)
    rows = []
    for sp in ("topr", "randomr"):
        for im, name in ((4, "p0"), (5, "p1"), (6, "p2")):
            for eps in grid:
                vol = err = 0.0
                for s in range(seeds):
                    g = normal_f32(hash64(s, hash64(0x5EED, seed)), dim)
                    sup = (ref.top_r(g, r) if sp == "topr" else random_r(dim, r, hash64(s, hash64(0x9AA9, seed))))
                    sup = np.asarray(sup, np.uint32)
                    target = np.zeros(dim, np.float32)
                    target[sup] = g[sup]
                    cfg = GpConfig.make(im, 0, fpr=eps, seed=hash64(s, hash64(0xC4A0, seed)))
                    c = ref.compress_pack(dim, sup, cfg, values=target[sup].astype(np.float64))
                    vol += ref.volume(c)["ratio_dense"]
                    _, dsup, dval = ref.decode(c)
                    dec = np.zeros(dim, np.float64)
                    dec[dsup.astype(np.int64)] = dval
                    t64 = target.astype(np.float64)
                    err += float(np.linalg.norm(dec - t64) / np.linalg.norm(t64))
                rows.append((sp, name, eps, vol / seeds, err / seeds))
    assert len(got) == len(rows)
    for line, (sp, name, eps, vol, err) in zip(got, rows):
        f = line.split(",")
        assert (f[0], f[1], float(f[2])) == (sp, name, eps)
        assert float(f[3]) == vol
        assert abs(float(f[4]) - err) <= 1e-12 * max(1.0, err)


def test_method_bench_rows():
    from paper_2102_03112_b200 import Codec
    from paper_2102_03112_b200.drivers import BENCH_ROWS, method_bench
    codec = Codec(max_d=200_000)
    lines = method_bench(200_000, 0.01, reps=2, fpr=0.01, seed=3, codec=codec).strip().splitlines()
    codec.close()
    assert lines[0] == "method,bits_total,t_encode_ns,t_decode_ns"
    names = [ln.split(",")[0] for ln in lines[1:]]
    assert names == [r[0] for r in BENCH_ROWS]
    for ln in lines[1:]:
        f = ln.split(",")
        assert int(f[1]) > 0 and int(f[2]) > 0 and int(f[3]) > 0, ln


@pytest.mark.parametrize("args,im,vm,kw", [(["--index", "bitmap"], 1, 0, {}), (["--policy", "p2", "--fpr", "0.001"], 6, 0,
                                                                                dict(fpr=0.001)),
                                           (["--index", "huffman", "--value", "quant", "--bits", "5"], 3, 3,
                                            dict(quant_bits=5)),
                                           (["--index", "rle", "--value", "deflate-slot", "--codec", "store"], 2, 4,
                                            dict(slot_codec=0))])
def test_cli_compress_decompress(tmp_path, oracle, args, im, vm, kw):
    """cmd_compress / cmd_decompress: the container file equals the oracle's
    compress of the same tensor; the decompressed tensor equals to_dense."""
    from oracle.bindings import GpConfig, synthetic_gradient
    from paper_2102_03112_b200.cli import main, read_tensor, write_tensor
    from paper_2102_03112_b200.dp import ratio_r
    d = 30_000
    g = synthetic_gradient(d, rank=3)
    write_tensor(str(tmp_path / "g.drt"), g)
    assert main(["compress", str(tmp_path / "g.drt"), str(tmp_path / "g.drc"), *args, "--topr", "0.01",
                 "--seed", "7"]) == 0
    c = (tmp_path / "g.drc").read_bytes()
    assert c == oracle.encode_dense(g, ratio_r(d, 0.01), GpConfig.make(im, vm, seed=7, **kw))
    assert main(["decompress", str(tmp_path / "g.drc"), str(tmp_path / "out.drt")]) == 0
    _, sup, val = oracle.decode(c)
    want = np.zeros(d, np.float32)
    want[sup.astype(np.int64)] = val.astype(np.float32)
    assert np.array_equal(read_tensor(str(tmp_path / "out.drt")), want)


def test_cli_decompress_reference_deflate(tmp_path, reference):
    """cmd_decompress of a container the reference wrote with its default codec (Deflate)."""
    from oracle.bindings import GpConfig, synthetic_gradient
    from paper_2102_03112_b200.cli import main, read_tensor
    d = 30_000
    g = synthetic_gradient(d, rank=5)
    c = reference.encode_dense(g, 300, GpConfig.make(1, 4, seed=7, slot_codec=1))
    (tmp_path / "g.drc").write_bytes(c)
    assert main(["decompress", str(tmp_path / "g.drc"), str(tmp_path / "out.drt")]) == 0
    _, sup, val = reference.decode(c)
    want = np.zeros(d, np.float32)
    want[sup.astype(np.int64)] = val.astype(np.float32)
    assert np.array_equal(read_tensor(str(tmp_path / "out.drt")), want)
