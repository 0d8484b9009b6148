"""Loaders for the committed golden fixtures (tests/golden/*.npz).

The fixtures were produced by running the reference gZCCL package
(tests/golden/make_golden.py); nothing here reads /root/reference.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _unpack(z, prefix):
    flat, offs = z[prefix + "_flat"], z[prefix + "_offs"]
    return [flat[offs[i] : offs[i + 1]] for i in range(len(offs) - 1)]


@dataclass
class CodecCase:
    name: str
    x: np.ndarray
    eb: float
    blob: bytes
    block_offsets: np.ndarray
    y: np.ndarray


def codec_cases():
    z = np.load(os.path.join(GOLDEN_DIR, "codec_cases.npz"))
    xs, blobs, offs, ys = _unpack(z, "x"), _unpack(z, "blob"), _unpack(z, "boffs"), _unpack(z, "y")
    return [CodecCase(str(z["names"][i]), xs[i].astype(np.float32), float(z["ebs"][i]), blobs[i].tobytes(), offs[i], ys[i])
            for i in range(len(xs))]


@dataclass
class RingCase:
    algo: str
    N: int
    n: int
    op: str
    eb: float
    inputs: list
    outputs: list
    msgs: list
    src: np.ndarray
    dst: np.ndarray


def ring_cases():
    z = np.load(os.path.join(GOLDEN_DIR, "ring_cases.npz"))
    out = []
    for k in range(int(z["count"])):
        p = f"c{k}_"
        N, n, ismax = (int(v) for v in z[p + "meta"])
        out.append(RingCase(str(z[p + "algo"]), N, n, "max" if ismax else "sum", float(z[p + "eb"]), _unpack(z, p + "in"),
                            _unpack(z, p + "out"), [m.tobytes() for m in _unpack(z, p + "msg")], z[p + "msg_src"], z[p + "msg_dst"]))
    return out


@dataclass
class ScatterCase:
    N: int
    root: int
    counts: list | None
    data: np.ndarray
    outputs: list
    msgs: list
    src: np.ndarray
    dst: np.ndarray


def scatter_cases():
    z = np.load(os.path.join(GOLDEN_DIR, "scatter_cases.npz"))
    out = []
    for k in range(int(z["count"])):
        p = f"s{k}_"
        N, root = (int(v) for v in z[p + "meta"])
        counts = [int(c) for c in z[p + "counts"]] or None
        out.append(ScatterCase(N, root, counts, z[p + "data"], _unpack(z, p + "out"), [m.tobytes() for m in _unpack(z, p + "msg")],
                               z[p + "msg_src"], z[p + "msg_dst"]))
    return out


def digests():
    with open(os.path.join(GOLDEN_DIR, "digests.json")) as f:
        return json.load(f)


def golden_blob(seed: int) -> bytes:
    with open(os.path.join(GOLDEN_DIR, f"blob_seed{seed}.bin"), "rb") as f:
        return f.read()


GOLDEN_CASES = {1: (1000, 1e-3), 2: (4096, 1e-4), 3: (31, 1e-5)}  # pkg/tests/conftest.py:7


def golden_data(seed):
    """pkg/tests/conftest.py:10-13."""
    n, eb = GOLDEN_CASES[seed]
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, n).astype(np.float32), eb


def fixed_rate_cases():
    """(x, bits, blob bytes, decoded y) from the reference's fixed_rate_compress."""
    z = np.load(os.path.join(GOLDEN_DIR, "fixed_rate_cases.npz"))
    xs, blobs, ys = _unpack(z, "x"), _unpack(z, "blob"), _unpack(z, "y")
    return [(xs[k], int(z["bits"][k]), blobs[k].tobytes(), ys[k]) for k in range(int(z["count"]))]


def fixed_rate_zero_cases():
    """Fixed-rate blobs whose min / max is a signed zero (numpy's AVX-512 choice)."""
    z = np.load(os.path.join(GOLDEN_DIR, "fixed_rate_zero_cases.npz"))
    xs, blobs, ys = _unpack(z, "x"), _unpack(z, "blob"), _unpack(z, "y")
    return [(xs[k], int(z["bits"][k]), blobs[k].tobytes(), ys[k]) for k in range(int(z["count"]))]
