"""The reference CLI's container subcommands on the device path
(tools/gradpack_main.cpp; tensor files: tensor_file.cpp:13-63, FORMAT.md "Tensor file").

  python -m paper_2102_03112_b200.cli compress IN.drt OUT.drc [--index M | --policy P] [--value V]
        [--fpr E] [--pd leftmost|middle|rightmost] [--degree K] [--segments S] [--bits B] [--bucket N]
        [--codec store|deflate] [--unsafe-naive] [--topr R] [--seed X]
  python -m paper_2102_03112_b200.cli decompress IN.drc OUT.drt
  python -m paper_2102_03112_b200.cli sweep|bench ...   (drivers.py)

compress: read_tensor → sparsify_ratio (R >= 1 keeps everything, else top_r of
llround(R*d)) → compress_gradient(sg, cfg, &g) + pack on the GPU → write, then
re-read, decode and report volume() as cmd_compress does (:182-209).
decompress: unpack + decompress_gradient + to_dense on the GPU → write_tensor.
The "train" subcommand (the SGD simulation harness) is outside this path.
"""
from __future__ import annotations

import argparse
import struct
import sys

import numpy as np

INDEX_NAMES = {"none": 0, "bitmap": 1, "rle": 2, "huffman": 3, "bloom-p0": 4, "bloom-p1": 5, "bloom-p2": 6,
               "bloom-pd": 7, "bloom-naive": 8}
POLICY_NAMES = {"p0": 4, "p1": 5, "p2": 6, "pd": 7, "naive": 8}
VALUE_NAMES = {"none": 0, "fit-poly": 1, "fit-dexp": 2, "quant": 3, "deflate-slot": 4, "raw-f64": 5}
PD_NAMES = {"leftmost": 0, "middle": 1, "rightmost": 2}
CODEC_NAMES = {"store": 0, "deflate": 1}


class TensorFileError(Exception):
    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


def tensor_to_bytes(g: np.ndarray) -> bytes:
    """tensor_to_bytes (tensor_file.cpp:13-20): "DRT1", u64 d, f32[d] LE."""
    g = np.ascontiguousarray(g, dtype="<f4")
    if g.size < 1:
        raise TensorFileError("Error", "tensor: dim must be >= 1")
    return b"DRT1" + struct.pack("<Q", g.size) + g.tobytes()


def tensor_from_bytes(b: bytes) -> np.ndarray:
    """tensor_from_bytes (tensor_file.cpp:22-33), same error classes and order."""
    if len(b) < 4:
        raise TensorFileError("TruncatedError", "byte stream exhausted")
    if b[:4] != b"DRT1":
        raise TensorFileError("DecodeError", "tensor: bad magic")
    if len(b) < 12:
        raise TensorFileError("TruncatedError", "byte stream exhausted")
    d = struct.unpack("<Q", b[4:12])[0]
    if d < 1:
        raise TensorFileError("CorruptPayloadError", "tensor: dim must be >= 1")
    if len(b) - 12 != 4 * d:
        raise TensorFileError("TruncatedError", "tensor: value section size mismatch")
    return np.frombuffer(b, dtype="<f4", offset=12, count=d).astype(np.float32)


def read_tensor(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        return tensor_from_bytes(f.read())


def write_tensor(path: str, g: np.ndarray) -> None:
    with open(path, "wb") as f:
        f.write(tensor_to_bytes(g))


def _config(a):
    from .api import PipelineConfig
    im = POLICY_NAMES[a.policy] if a.policy else INDEX_NAMES[a.index]
    if im == 8 and not a.unsafe_naive:
        raise SystemExit("error: --index bloom-naive misaligns values by design; pass --unsafe-naive")
    return PipelineConfig(index_method=im, value_method=VALUE_NAMES[a.value], fpr=a.fpr, pd_variant=PD_NAMES[a.pd],
                          degree=a.degree, max_segments=a.segments, quant_bits=a.bits, quant_bucket=a.bucket,
                          slot_codec=CODEC_NAMES[a.codec], seed=a.seed)


def cmd_compress(a) -> int:
    import torch

    from .api import Codec, volume
    from .dp import ratio_r
    cfg = _config(a)
    sys.stderr.write(f"config: subcommand=compress input={a.input} output={a.output} index={a.policy or a.index} "
                     f"value={a.value} fpr={a.fpr} topr={a.topr} seed={a.seed}\n")
    g = read_tensor(a.input)
    d = g.size
    r = d if a.topr >= 1.0 else ratio_r(d, a.topr)  # sparsify_ratio (gradpack_main.cpp:168-173)
    codec = Codec(max_d=d)
    c = codec.compress(torch.from_numpy(g).cuda(), r, cfg).cpu().numpy().tobytes()
    with open(a.output, "wb") as f:
        f.write(c)
    with open(a.output, "rb") as f:  # validate what landed on disk (:187-189)
        back = f.read()
    codec.decompress(torch.from_numpy(np.frombuffer(back, np.uint8).copy()).cuda())
    v = volume(back)
    print(f"d={d} r={int.from_bytes(back[17:25], 'little')}")
    print(f"volume: index_bits={v['index_bits']} value_bits={v['value_bits']} reorder_bits={v['reorder_bits']} "
          f"metadata_bits={v['metadata_bits']} total_bits={v['total_bits']} ratio_dense={v['ratio_dense']:.6g} "
          f"ratio_sparse={v['ratio_sparse']:.6g}")
    print(f"wrote {a.output} ({(v['total_bits'] + 7) // 8} bytes)")
    codec.close()
    return 0


def cmd_decompress(a) -> int:
    import torch

    from .api import Codec
    sys.stderr.write(f"config: subcommand=decompress input={a.input} output={a.output}\n")
    with open(a.input, "rb") as f:
        c = f.read()
    if len(c) < 49:
        raise SystemExit("error: byte stream exhausted")
    d = int.from_bytes(c[9:17], "little")
    codec = Codec(max_d=max(1, d))
    dense = torch.zeros(d, dtype=torch.float32, device="cuda")
    codec.decode_accumulate(torch.from_numpy(np.frombuffer(c, np.uint8).copy()).cuda(), dense, scale=1.0)
    codec.status()
    write_tensor(a.output, dense.cpu().numpy())
    read_tensor(a.output)
    print(f"wrote {a.output} (d={d})")
    codec.close()
    return 0


def main(argv=None) -> int:
    from . import drivers
    ap = argparse.ArgumentParser(prog="python -m paper_2102_03112_b200.cli")
    sub = ap.add_subparsers(dest="cmd", required=True)
    co = sub.add_parser("compress", help="tensor file (.drt) -> container (.drc)")
    co.add_argument("input")
    co.add_argument("output")
    co.add_argument("--index", default="bitmap", choices=sorted(INDEX_NAMES))
    co.add_argument("--policy", choices=sorted(POLICY_NAMES))
    co.add_argument("--value", default="none", choices=sorted(VALUE_NAMES))
    co.add_argument("--fpr", type=float, default=0.01)
    co.add_argument("--pd", default="leftmost", choices=sorted(PD_NAMES))
    co.add_argument("--degree", type=int, default=5)
    co.add_argument("--segments", type=int, default=0)
    co.add_argument("--bits", type=int, default=7)
    co.add_argument("--bucket", type=int, default=512)
    co.add_argument("--codec", default="deflate", choices=sorted(CODEC_NAMES))
    co.add_argument("--unsafe-naive", action="store_true")
    co.add_argument("--topr", type=float, default=1.0)
    co.add_argument("--seed", type=int, default=1)
    de = sub.add_parser("decompress", help="container (.drc) -> tensor file (.drt)")
    de.add_argument("input")
    de.add_argument("output")
    for name in ("sweep", "bench"):
        sub.add_parser(name, add_help=False)
    a, rest = ap.parse_known_args(argv)
    try:
        if a.cmd == "compress":
            return cmd_compress(a)
        if a.cmd == "decompress":
            return cmd_decompress(a)
        return drivers.main([a.cmd, *rest])
    except (TensorFileError, RuntimeError) as e:
        sys.stderr.write(f"error: {e}\n")
        return 1


if __name__ == "__main__":
    raise SystemExit(main())
