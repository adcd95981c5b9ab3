"""Reference file formats for the STL hot path.

Byte-compatible readers and writers for the reference's blobs, so triples and layers trained
or encoded by the reference load straight onto the GPU path and GPU results can be dumped
for offline parity:

=============================  ==========================================  =====================
reference (file:line)          format                                      here
=============================  ==========================================  =====================
dense_core.py:170-232          STLM matrix blob: "STLM", u32 version,      matrix_to_bytes /
                               u64 rows, u64 cols, f64 data (LE); CSV      matrix_from_bytes, CSV
snf_operator.py:191-228        SnfTriple: JSON header line {"t","r",       triple_to_bytes /
                               "version"} + STLM e_x, e_w, d               triple_from_bytes
snf_operator.py:231-257        STLE encoded tensor: "STLE", u32 version,   encoded_to_bytes /
                               u64 R, C, r, f64 fibers (r contiguous)      encoded_from_bytes
toy_network.py:348-380         model checkpoint: JSON header {"version",   save_model /
                               "segments"} + per layer triple + STLE        load_model
=============================  ==========================================  =====================

Host-side byte handling only (numpy); no compute. Tensors given as GPU planes are brought to the
host and converted to the reference's fiber-contiguous layout (encoded (R, C, r), weights
(K/t, N/t, r)). Factors of a loaded SnfTriple are held in fp32 (the compute precision): a blob
round-trips byte-for-byte when its values are fp32-exact (e.g. Strassen factors, fp32 data).
"""

from __future__ import annotations

import json
import struct
from pathlib import Path

import numpy as np

from .dense_core import ShapeError

MATRIX_MAGIC = b"STLM"
MATRIX_VERSION = 1
ENCODED_MAGIC = b"STLE"
ENCODED_VERSION = 1
TRIPLE_VERSION = 1
MODEL_VERSION = 1


def _f64(a) -> np.ndarray:
    """numpy / torch (any device, any float dtype) -> C-contiguous float64 numpy."""
    if hasattr(a, "detach"):
        a = a.detach().to("cpu").double().numpy()
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _matrix(a, name: str = "matrix") -> np.ndarray:
    m = _f64(a)
    if m.ndim != 2:
        raise ShapeError(f"{name} must be 2-D, got ndim={m.ndim}")
    if m.size and not np.isfinite(m).all():
        raise ValueError(f"{name} contains non-finite entries")
    return m


# ------------------------------------------------------------------ matrices (dense_core.py)
def matrix_to_bytes(m) -> bytes:
    """dense_core.py:206-209."""
    m = _matrix(m)
    return MATRIX_MAGIC + struct.pack("<IQQ", MATRIX_VERSION, *m.shape) + m.astype("<f8").tobytes()


def matrix_from_bytes(buf: bytes, offset: int = 0) -> tuple[np.ndarray, int]:
    """dense_core.py:212-224: one matrix blob at `offset` -> (matrix, next offset)."""
    head = offset + 4 + 4 + 8 + 8
    if len(buf) < head or buf[offset:offset + 4] != MATRIX_MAGIC:
        raise ValueError("not a matrix blob (bad magic or truncated header)")
    version, rows, cols = struct.unpack_from("<IQQ", buf, offset + 4)
    if version != MATRIX_VERSION:
        raise ValueError(f"unsupported matrix blob version {version}")
    end = head + rows * cols * 8
    if len(buf) < end:
        raise ValueError("truncated matrix blob payload")
    data = np.frombuffer(buf[head:end], dtype="<f8").reshape(rows, cols).copy()
    return _matrix(data), end


def save_matrix_blob(path, m) -> None:
    Path(path).write_bytes(matrix_to_bytes(m))


def load_matrix_blob(path) -> np.ndarray:
    return matrix_from_bytes(Path(path).read_bytes())[0]


def matrix_to_csv(m) -> str:
    """dense_core.py:177-179: one row per line, shortest round-trip float text."""
    m = _matrix(m)
    return "\n".join(",".join(repr(x) for x in row) for row in m.tolist()) + "\n"


def matrix_from_csv(text: str) -> np.ndarray:
    """dense_core.py:182-194 (blank lines and '#' comments skipped)."""
    rows = []
    for line in text.splitlines():
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        rows.append([float(tok) for tok in line.split(",")])
    if not rows:
        raise ValueError("no matrix rows found in CSV text")
    if any(len(r) != len(rows[0]) for r in rows):
        raise ShapeError("ragged CSV rows")
    return _matrix(np.array(rows))


def save_matrix_csv(path, m) -> None:
    Path(path).write_text(matrix_to_csv(m))


def load_matrix_csv(path) -> np.ndarray:
    return matrix_from_csv(Path(path).read_text())


# ------------------------------------------------------------------ triples (snf_operator.py)
def triple_to_bytes(snf) -> bytes:
    """snf_operator.py:199-206: JSON header line + e_x, e_w, d matrix blobs."""
    header = json.dumps({"t": int(snf.t), "r": int(snf.r), "version": TRIPLE_VERSION}) + "\n"
    return (header.encode() + matrix_to_bytes(snf.e_x) + matrix_to_bytes(snf.e_w)
            + matrix_to_bytes(snf.d))


def triple_from_bytes(buf: bytes):
    """snf_operator.py:209-220 -> SnfTriple (fp32 factors, on the host until first use)."""
    from .snf_operator import SnfTriple

    nl = buf.find(b"\n")
    if nl < 0:
        raise ValueError("triple blob has no header line")
    header = json.loads(buf[:nl].decode())
    if header.get("version") != TRIPLE_VERSION:
        raise ValueError(f"unsupported triple version {header.get('version')}")
    offset = nl + 1
    e_x, offset = matrix_from_bytes(buf, offset)
    e_w, offset = matrix_from_bytes(buf, offset)
    d, offset = matrix_from_bytes(buf, offset)
    return SnfTriple(int(header["t"]), int(header["r"]), e_x, e_w, d)


def save_triple(path, snf) -> None:
    Path(path).write_bytes(triple_to_bytes(snf))


def load_triple(path):
    return triple_from_bytes(Path(path).read_bytes())


# ------------------------------------------------------------------ encoded tensors (STLE)
def _encoded(enc) -> np.ndarray:
    e = _f64(enc)
    if e.ndim != 3:
        raise ShapeError("encoded tensor must be a (block_rows, block_cols, r) tensor")
    return e


def encoded_to_bytes(enc) -> bytes:
    """snf_operator.py:231-234. `enc` in the reference layout (R, C, r) — the reference-shaped
    views this package returns (e.g. ``encode_tiles``, ``StlLayer.weights``) qualify."""
    e = _encoded(enc)
    return ENCODED_MAGIC + struct.pack("<IQQQ", ENCODED_VERSION, *e.shape) + e.astype("<f8").tobytes()


def encoded_from_bytes(buf: bytes, offset: int = 0) -> tuple[np.ndarray, int]:
    """snf_operator.py:237-249 -> ((R, C, r) float64, next offset)."""
    head = offset + 4 + 4 + 24
    if len(buf) < head or buf[offset:offset + 4] != ENCODED_MAGIC:
        raise ValueError("not an encoded-tiles blob")
    version, br, bc, r = struct.unpack_from("<IQQQ", buf, offset + 4)
    if version != ENCODED_VERSION:
        raise ValueError(f"unsupported encoded-tiles version {version}")
    end = head + br * bc * r * 8
    if len(buf) < end:
        raise ValueError("truncated encoded-tiles blob")
    data = np.frombuffer(buf[head:end], dtype="<f8").reshape(br, bc, r).copy()
    return data, end


def save_encoded(path, enc) -> None:
    Path(path).write_bytes(encoded_to_bytes(enc))


def load_encoded(path) -> np.ndarray:
    return encoded_from_bytes(Path(path).read_bytes())[0]


# ------------------------------------------------------------------ model checkpoints
def model_to_bytes(layers) -> bytes:
    """toy_network.py:351-361. `layers`: StlLayer objects or (snf, weights) pairs with weights
    in the reference layout (in_tiles, out_tiles, r)."""
    segments, payload = [], b""
    for layer in layers:
        snf, weights = (layer.snf, layer.weights) if hasattr(layer, "snf") else layer
        tb, eb = triple_to_bytes(snf), encoded_to_bytes(weights)
        segments.append([len(tb), len(eb)])
        payload += tb + eb
    header = json.dumps({"version": MODEL_VERSION, "segments": segments}) + "\n"
    return header.encode() + payload


def model_from_bytes(buf: bytes):
    """toy_network.py:364-380 -> [(SnfTriple, weights (in_tiles, out_tiles, r) float64)]."""
    nl = buf.find(b"\n")
    if nl < 0:
        raise ValueError("model checkpoint has no header line")
    header = json.loads(buf[:nl].decode())
    if header.get("version") != MODEL_VERSION:
        raise ValueError(f"unsupported model checkpoint version {header.get('version')}")
    out, offset = [], nl + 1
    for t_len, e_len in header["segments"]:
        snf = triple_from_bytes(buf[offset:offset + t_len])
        offset += t_len
        weights, _ = encoded_from_bytes(buf[offset:offset + e_len])
        offset += e_len
        if weights.shape[2] != snf.r:
            raise ShapeError(f"layer weights rank {weights.shape[2]} != triple rank {snf.r}")
        out.append((snf, weights))
    return out


def save_model(path, layers) -> None:
    Path(path).write_bytes(model_to_bytes(layers))


def load_model(path, dtype=None, device=None):
    """Checkpoint -> list of GPU ``StlLayer`` (weights as slice-major planes in `dtype`,
    default fp32)."""
    import torch

    from .dense_core import default_device
    from .layer import StlLayer

    dev = device if device is not None else default_device()
    layers = []
    for snf, w in model_from_bytes(Path(path).read_bytes()):
        wt = torch.from_numpy(w).to(device=dev, dtype=dtype or torch.float32)
        layers.append(StlLayer(snf.to(dev), wt))
    return layers
