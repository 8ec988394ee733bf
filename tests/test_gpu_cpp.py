"""The C++ drop-in (include/gradpack_b200.hpp) driven from a C++ host program,
checked against the oracle: container bytes, decoded supports/values, and the
exception class a gradpack C++ caller would catch for a corrupt container."""
import os
import struct
import subprocess

import numpy as np
import pytest

from oracle.bindings import GpConfig, synthetic_gradient

pytestmark = pytest.mark.gpu

CLI = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "gp_cli")


def _run(args):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=120)


@pytest.mark.parametrize("im,vm,fpr", [(1, 0, 0.01), (2, 0, 0.01), (6, 0, 0.001), (5, 5, 0.01), (0, 0, 0.01)])
def test_cpp_encode_matches_oracle(tmp_path, oracle, im, vm, fpr):
    g = synthetic_gradient(300_000, rank=7)
    gp = tmp_path / "g.f32"
    g.tofile(gp)
    out = tmp_path / "c.drc"
    res = _run(["encode", gp, 3000, im, vm, fpr, 42, out])
    assert res.returncode == 0, res.stderr
    assert out.read_bytes() == oracle.encode_dense(g, 3000, GpConfig.make(im, vm, fpr=fpr, seed=42))
    assert f"bytes={out.stat().st_size}" in res.stdout


def test_cpp_decode_and_errors(tmp_path, oracle):
    g = synthetic_gradient(100_000, rank=3)
    c = oracle.encode_dense(g, 1000, GpConfig.make(6, 1, fpr=0.01, seed=5))
    cp = tmp_path / "c.drc"
    cp.write_bytes(c)
    res = _run(["decode", cp, tmp_path / "s.u32", tmp_path / "v.f64"])
    assert res.returncode == 0, res.stderr
    _, sup, val = oracle.decode(c)
    assert np.array_equal(np.fromfile(tmp_path / "s.u32", np.uint32), sup)
    assert np.array_equal(np.fromfile(tmp_path / "v.f64", np.float64), val)
    # corrupt: flip a payload byte → ChecksumError (exit 10 + GP_CHECKSUM)
    bad = bytearray(c)
    bad[60] ^= 1
    cp.write_bytes(bytes(bad))
    assert _run(["decode", cp, tmp_path / "s", tmp_path / "v"]).returncode == 10 + 4
    # truncated
    cp.write_bytes(c[:30])
    assert _run(["decode", cp, tmp_path / "s", tmp_path / "v"]).returncode == 10 + 3
    # unknown index method with a valid CRC → UnknownMethodError
    bad = bytearray(c)
    bad[6] = 11
    cp.write_bytes(bytes(bad))
    assert _run(["decode", cp, tmp_path / "s", tmp_path / "v"]).returncode == 10 + 5
    assert struct.unpack_from("<Q", c, 9)[0] == 100_000
