"""Router-bank wire format (`.bank`, magic TIDE v1) -> host + device router cache.

Byte-compatible with the reference's `save_bank` / `load_bank`
(ee/calibration.py:418-497, layout pkg/docs/file_formats.md:30-70) and its
container checks (ee/_binio.py): a load validates magic, version, field
plausibility, total size, CRC32, then the payload, raising the same error
classes (`BadMagicError`, `VersionError`, `DimensionError`, `TruncatedError`,
`ChecksumError`, all `BinaryFormatError`) with the same message substrings.

What changes is where the bytes go.  The file is read once into one host
buffer (page-locked when a device is requested); every router's W_down /
w_up are zero-copy f32 views of it; with `device=` the whole payload crosses
PCIe in ONE copy and the kernel-dtype W_down copies (bf16 / f16 for the
tensor-core route, f32 for the CUDA-core path) are cut from it on the device
and installed in the router weight cache, so the first routed batch finds
them resident.
"""

from __future__ import annotations

import os
import struct
import zlib

import numpy as np
import torch

from . import _native as N
from . import router_ops as R
from .calibration import BANK_MAGIC, BANK_VERSION, RouterBank, RouterStats
from .router_ops import Router

_HEADER = 44  # magic .. model digest (file_formats.md:38-52)
_REC_HEAD = 24  # layer, examples, positives, flags, final_loss, accuracy


class BinaryFormatError(Exception):
    """Base class for malformed container files (ee/_binio.py:17)."""


class BadMagicError(BinaryFormatError):
    pass


class VersionError(BinaryFormatError):
    pass


class TruncatedError(BinaryFormatError):
    pass


class ChecksumError(BinaryFormatError):
    pass


class DimensionError(BinaryFormatError):
    pass


def bank_file_size(hidden_dim: int, bottleneck: int, n_checkpoints: int) -> int:
    """Exact on-disk size in bytes (ee/calibration.py:418-422)."""
    return _HEADER + n_checkpoints * (_REC_HEAD + 4 * (bottleneck * hidden_dim + bottleneck)) + 4


def save_bank(bank, path) -> None:
    """Write `bank` in the reference's layout (ee/calibration.py:425-446).

    Accepts this package's RouterBank or the reference's (duck-typed)."""
    parts = [BANK_MAGIC, struct.pack("<IIIIffIIQ", BANK_VERSION, bank.hidden_dim,
                                     bank.bottleneck, bank.interval, bank.tau, bank.eps,
                                     bank.num_layers, len(bank.routers), bank.model_digest)]
    for k in bank.checkpoints:
        router, st = bank.routers[k], bank.stats[k]
        parts.append(struct.pack("<IIIIff", k, st.examples, st.positives, st.flags,
                                 st.final_loss, st.accuracy))
        parts.append(np.ascontiguousarray(router.w_down, dtype="<f4").tobytes())
        parts.append(np.ascontiguousarray(router.w_up, dtype="<f4").tobytes())
    body = b"".join(parts)
    with open(path, "wb") as fh:
        fh.write(body)
        fh.write(struct.pack("<I", zlib.crc32(body) & 0xFFFFFFFF))


def _read_file(path, pinned: bool):
    size = os.path.getsize(path)
    if pinned and size > 0:
        buf_t = torch.empty(size, dtype=torch.uint8, pin_memory=True)
        buf = buf_t.numpy()
    else:
        buf_t = None
        buf = np.empty(size, dtype=np.uint8)
    with open(path, "rb") as fh:
        got = fh.readinto(memoryview(buf))
    if got != size:
        raise TruncatedError(f"short read: {got} of {size} bytes")
    return buf, buf_t


def _parse(buf: np.ndarray):
    """Validate in the reference's order; -> (meta tuple, record offsets)."""
    data = memoryview(buf)
    n = len(data)
    if n < 8:
        raise TruncatedError(f"container holds {n} bytes, too short for any header")
    limit = n - 4  # the CRC trailer is never part of a field

    def take(pos, size):
        if pos + size > limit:
            raise TruncatedError(
                f"needed {size} bytes at offset {pos}, only {limit - pos} before trailer")
        return data[pos:pos + size]

    magic = bytes(take(0, 4))
    if magic != BANK_MAGIC:
        raise BadMagicError(f"bad magic {magic!r}, expected {BANK_MAGIC!r}")
    (version,) = struct.unpack("<I", take(4, 4))
    if version != BANK_VERSION:
        raise VersionError(f"unsupported bank version {version}")
    d, b, interval = struct.unpack("<III", take(8, 12))
    tau, eps = struct.unpack("<ff", take(20, 8))
    num_layers, n_ckpt = struct.unpack("<II", take(28, 8))
    (digest,) = struct.unpack("<Q", take(36, 8))
    if d < 1 or b < 1 or interval < 1 or num_layers < 2:
        raise DimensionError(
            f"implausible bank metadata: d={d}, b={b}, c={interval}, L={num_layers}")
    if n_ckpt < 1 or n_ckpt > num_layers:
        raise DimensionError(f"bank declares {n_ckpt} checkpoints for {num_layers} layers")
    expected = bank_file_size(d, b, n_ckpt)
    if n < expected:
        raise TruncatedError(f"file holds {n} bytes, metadata implies {expected}")
    if n > expected:
        raise DimensionError(
            f"file holds {n} bytes but metadata implies {expected}; trailing data")
    (stored,) = struct.unpack("<I", data[n - 4:n])
    computed = zlib.crc32(data[:n - 4]) & 0xFFFFFFFF
    if stored != computed:
        raise ChecksumError(f"CRC32 mismatch: stored {stored:#010x}, computed {computed:#010x}")
    rec = _REC_HEAD + 4 * (b * d + b)
    offs = [_HEADER + i * rec for i in range(n_ckpt)]
    return (d, b, interval, tau, eps, num_layers, digest), offs


def load_bank(path, *, device=None, dtype=None) -> RouterBank:
    """Read a `.bank` file (ee/calibration.py:449-497).

    device: optional CUDA device — the payload is copied there once and each
    router's W_down is installed in the device weight cache in `dtype`
    (torch.bfloat16 default, torch.float16 or torch.float32)."""
    buf, buf_t = _read_file(path, pinned=device is not None)
    (d, b, interval, tau, eps, num_layers, digest), offs = _parse(buf)
    routers, stats = {}, {}
    previous = -1
    for off in offs:
        layer, examples, positives, flags = struct.unpack_from("<IIII", buf, off)
        final_loss, accuracy = struct.unpack_from("<ff", buf, off + 16)
        if layer <= previous or layer >= num_layers:
            raise DimensionError(
                f"checkpoint layer {layer} out of order or beyond layer count {num_layers}")
        previous = layer
        w0 = off + _REC_HEAD
        w_down = buf[w0:w0 + 4 * b * d].view("<f4").reshape(b, d)
        w_up = buf[w0 + 4 * b * d:w0 + 4 * (b * d + b)].view("<f4").reshape(1, b)
        routers[layer] = Router(layer=layer, w_down=w_down, w_up=w_up)
        stats[layer] = RouterStats(examples=examples, positives=positives,
                                   final_loss=final_loss, accuracy=accuracy, flags=flags)
    bank = RouterBank(hidden_dim=d, bottleneck=b, interval=interval, tau=tau, eps=eps,
                      num_layers=num_layers, model_digest=digest, routers=routers, stats=stats)
    if device is not None:
        install_device_weights(bank, device, dtype or torch.bfloat16, buf_t, offs)
    return bank


_CODES = {torch.bfloat16: N.BF16, torch.float16: N.F16, torch.float32: N.F32}


def install_device_weights(bank, device, dtype, host_buf=None, offs=None) -> None:
    """Put every router's kernel-dtype W_down and f32 w_up on `device`.

    With the file buffer (`load_bank(device=...)`) the whole payload is one
    host->device copy; otherwise one copy per router."""
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ValueError("install_device_weights needs a CUDA device")
    if dtype not in _CODES:
        raise ValueError(f"unsupported router dtype {dtype}")
    code = _CODES[dtype]
    d, b = bank.hidden_dim, bank.bottleneck
    if host_buf is None:
        for k in bank.checkpoints:
            R.device_weights(bank.routers[k], code, dev)
        return
    payload = host_buf.to(dev, non_blocking=True)
    for k, off in zip(bank.checkpoints, offs):
        w0 = off + _REC_HEAD
        wd32 = payload[w0:w0 + 4 * b * d].view(torch.float32).view(b, d)
        wu = payload[w0 + 4 * b * d:w0 + 4 * (b * d + b)].view(torch.float32).clone()
        wd = wd32.to(dtype).contiguous() if dtype != torch.float32 else wd32.clone()
        R.install_cached(bank.routers[k], code, dev, wd, wu)
    torch.cuda.current_stream(dev).synchronize()  # the pinned buffer may be freed after return
