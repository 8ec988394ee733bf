"""Tensor files (.drt, tensor_file.cpp:13-33): round trip and the reference's
error classes, host-only."""
import struct

import numpy as np
import pytest

from paper_2102_03112_b200.cli import TensorFileError, tensor_from_bytes, tensor_to_bytes


def test_round_trip():
    g = np.random.default_rng(1).standard_normal(1001).astype(np.float32)
    b = tensor_to_bytes(g)
    assert b[:4] == b"DRT1" and struct.unpack("<Q", b[4:12])[0] == 1001 and len(b) == 12 + 4 * 1001
    assert np.array_equal(tensor_from_bytes(b), g)


@pytest.mark.parametrize("blob,kind", [(b"DR", "TruncatedError"), (b"XRT1" + bytes(12), "DecodeError"),
                                       (b"DRT1" + struct.pack("<Q", 0), "CorruptPayloadError"),
                                       (b"DRT1" + struct.pack("<Q", 3) + bytes(8), "TruncatedError"),
                                       (b"DRT1" + struct.pack("<Q", 1) + bytes(8), "TruncatedError")])
def test_errors(blob, kind):
    with pytest.raises(TensorFileError) as e:
        tensor_from_bytes(blob)
    assert e.value.kind == kind
