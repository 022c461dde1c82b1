"""Tensor codec and container of the drop-in API -- host side over libitq3.

Mirrors the reference interface (pkg/src/itq3/codec.py:57-291): same names, argument
meaning, validation order and error classes/messages.  The work runs in sm_100a kernels:
  quantize_tensor / encode_block   -> K1 ``itq3_encode``   (bit-exact container bytes)
  dequantize_tensor / decode_block -> K2 ``itq3_dequant``  (value-exact)
  read_container block checks      -> K7 ``itq3_validate`` (one pass, first offender)
A ``QuantizedTensor`` keeps its payload resident on the GPU in the container's byte order
(so ``write_container`` is a straight copy) plus, on first use by the fused kernels, the
tiled GEMV layout (``itq3_repack_tiled``).
"""

from __future__ import annotations

import io
import os
import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import (BadMagicError, ContainerError, CorruptionError, DomainError, LengthError, ShapeError,
                     SizeMismatchError, TruncatedStreamError, UnsupportedVersionError)
from .packing import PackedBlock, block_from_bytes, block_nbytes
from .quantizer import POLICY_CODE, ScalePolicy

MAGIC = b"ITQ3"
VERSION = 1
FLAG_SUB_SCALES = 0x1
FLAG_ASYMMETRIC = 0x2
KNOWN_FLAGS = FLAG_SUB_SCALES | FLAG_ASYMMETRIC
HEADER = struct.Struct("<4sHHQQII")  # magic, version, flags, rows, cols, block_n, pad (32 bytes)
BLOCK_SIZES = (32, 64, 128, 256, 512)
VARIANTS = ("s", "ss")
SUB_BLOCKS = 8


@dataclass(frozen=True)
class QuantConfig:
    """Encoder settings (codec.py:57-70)."""

    block_n: int = 256
    variant: str = "s"
    policy: ScalePolicy = field(default_factory=ScalePolicy)
    symmetric: bool = True

    def __post_init__(self):
        if self.block_n not in BLOCK_SIZES:
            raise DomainError(f"QuantConfig: block_n must be one of {BLOCK_SIZES}, got {self.block_n}")
        if self.variant not in VARIANTS:
            raise DomainError(f"QuantConfig: variant must be one of {VARIANTS}, got {self.variant!r}")


class QuantizedTensor:
    """A quantized matrix: header fields + device-resident block payload.

    Constructible like the reference dataclass (``blocks=`` list of PackedBlock) or from a
    device payload (``payload=`` uint8 CUDA tensor, n_blocks x block_nbytes).  ``blocks`` is
    materialised lazily from the payload (for equality / inspection / serialisation).
    """

    def __init__(self, rows: int, cols: int, block_n: int, variant: str, symmetric: bool, pad: int,
                 blocks: list | None = None, *, payload: torch.Tensor | None = None, validated: bool = False):
        self.rows, self.cols, self.block_n = int(rows), int(cols), int(block_n)
        self.variant, self.symmetric, self.pad = variant, bool(symmetric), int(pad)
        if (blocks is None) == (payload is None):
            raise ValueError("QuantizedTensor: give exactly one of blocks= or payload=")
        self._blocks = list(blocks) if blocks is not None else None
        self._payload = payload
        self._validated = validated  # planes + zero-point checked (decode paths)
        self._tiled = {}
        self._mmq = {}
        self._mmq8 = {}
        self._k5_range = None
        self._chain1 = {}  # device -> one-stage chain context of the k = 1 path (compute.py)

    # -- reference-compatible surface ------------------------------------------------------------
    @property
    def n_blocks(self) -> int:
        return -(-self.rows * self.cols // self.block_n)

    @property
    def bits_per_weight(self) -> float:
        return 8.0 * len(self) * self.block_nbytes / (self.rows * self.cols)

    def __len__(self) -> int:
        return len(self._blocks) if self._blocks is not None else int(self._payload.shape[0])

    @property
    def block_nbytes(self) -> int:
        return block_nbytes(self.block_n, self.variant == "ss")

    @property
    def blocks(self) -> list:
        if self._blocks is None:
            raw = self._payload.cpu().numpy()
            ss = self.variant == "ss"
            self._blocks = [block_from_bytes(raw[i].tobytes(), self.block_n, ss) for i in range(raw.shape[0])]
        return self._blocks

    def __eq__(self, other) -> bool:
        if not isinstance(other, QuantizedTensor):
            return NotImplemented
        head = (self.rows, self.cols, self.block_n, self.variant, self.symmetric, self.pad)
        if head != (other.rows, other.cols, other.block_n, other.variant, other.symmetric, other.pad):
            return False
        if self._payload is not None and other._payload is not None:
            a, b = self._payload, other._payload
            return a.shape == b.shape and bool(torch.equal(a, b.to(a.device)))
        return self.blocks == other.blocks

    def __repr__(self) -> str:
        return (f"QuantizedTensor(rows={self.rows}, cols={self.cols}, block_n={self.block_n}, "
                f"variant={self.variant!r}, symmetric={self.symmetric}, pad={self.pad}, n_blocks={len(self)})")

    # -- device residency ---------------------------------------------------------------------------
    def payload(self, dev=None) -> torch.Tensor:
        """Device payload (n_blocks, block_nbytes) uint8, uploaded from ``blocks`` if needed."""
        dev = dev or _lib.device()
        if self._payload is None:
            ss = self.variant == "ss"
            want = block_nbytes(self.block_n, ss)
            for i, blk in enumerate(self._blocks):
                if blk.n != self.block_n or (blk.sub_scale_bits is not None) != ss:
                    raise ShapeError(f"container: block {i} does not match block_n {self.block_n} / "
                                     f"variant {self.variant!r}")
            if len(self._blocks) != self.n_blocks:
                raise ShapeError(f"container: {len(self._blocks)} blocks, expected {self.n_blocks}")
            host = np.frombuffer(b"".join(b.to_bytes() for b in self._blocks), np.uint8).reshape(-1, want)
            self._payload = torch.from_numpy(host.copy()).to(dev)
        elif self._payload.device != dev:
            self._payload = self._payload.to(dev)
        return self._payload

    def ensure_decodable(self) -> torch.Tensor:
        """Payload after the decode-path checks (stored code <= 2, finite zero-point), cached."""
        p = self.payload()
        if not self._validated:
            validate_payload(p, self.block_n, self.variant == "ss", full=False, prefix=True)
            self._validated = True
        return p

    def fast_layout(self) -> bool:
        return self.block_n == 256 and self.variant == "s" and self.cols % 256 == 0

    def tiled(self) -> torch.Tensor:
        """Tiled GEMV/MMQ layout (csrc/gemv.cu) for the fast path, built once per device."""
        if len(self._tiled) == 1 and (self._payload is None or not self._payload.is_cuda):
            return next(iter(self._tiled.values()))
        p = self.ensure_decodable()
        key = p.device
        if key not in self._tiled:
            asym = 0 if self.symmetric else 1
            nbytes = _lib.load().itq3_tiled_nbytes(self.rows, self.cols, asym)
            t = torch.empty(nbytes, dtype=torch.uint8, device=p.device)
            _lib.call("itq3_repack_tiled", _lib.ptr(p), self.rows, self.cols, asym, _lib.ptr(t),
                      _lib.stream_ptr(p.device))
            self._tiled[key] = t
        return self._tiled[key]

    def mmq8_layout(self) -> torch.Tensor:
        """Small-batch tcgen05 i8 MMQ layout (csrc/mmq.cu K5b: 128-row x 256-k records)."""
        p = self.ensure_decodable()
        if p.device not in self._mmq8:
            asym = 0 if self.symmetric else 1
            t = torch.empty(_lib.load().itq3_mmq8_nbytes(self.rows, self.cols), dtype=torch.uint8, device=p.device)
            _lib.call("itq3_repack_mmq8", _lib.ptr(p), self.rows, self.cols, asym, _lib.ptr(t),
                      _lib.stream_ptr(p.device))
            self._mmq8[p.device] = t
        return self._mmq8[p.device]

    def mmq_ok(self) -> bool:
        """K5 (tcgen05 f16 MMQ) handles cols % 256 == 0 with whole blocks per row, every block_n
        (variant ss: block_n >= 256, whose sub-blocks are at least 32 wide)."""
        return (self.cols % 256 == 0 and self.cols % self.block_n == 0
                and (self.variant == "s" or self.block_n >= 256))

    def k5_range_ok(self) -> bool:
        """K5 forms A = d t in binary16: exact as long as |2 d| <= 65504, i.e. every stored scale (or
        sub-scale) magnitude is below 2^15 and finite.  Checked once per tensor on the device; a tensor
        with a larger scale takes a path with fp32 scales (K4 GEMV, or the exact generic kernel)."""
        if self._k5_range is None:
            p = self.ensure_decodable()
            q = 3 * self.block_n // 8
            lo, hi = (q + 4, q + 20) if self.variant == "ss" else (q, q + 2)
            bits = p.reshape(-1, p.shape[-1])[:, lo:hi].contiguous().view(torch.int16)
            self._k5_range = bool(((bits & 0x7FFF) <= 0x77FF).all()) if bits.numel() else True
        return self._k5_range

    def mmq_flags(self) -> int:
        """itq3_mmq* flags: ITQ3_MMQ_ASYM (1) | ITQ3_MMQ_PER32 (2: variant ss or block_n != 256)."""
        return (0 if self.symmetric else 1) | (2 if (self.variant == "ss" or self.block_n != 256) else 0)

    def mmq_layout(self) -> torch.Tensor:
        """tcgen05 MMQ layout (csrc/mmq.cu: 2-bit codes in 64-k slabs, rows padded to 128)."""
        p = self.ensure_decodable()
        if p.device not in self._mmq:
            flags = self.mmq_flags()
            t = torch.empty(_lib.load().itq3_mmq_nbytes(self.rows, self.cols, flags), dtype=torch.uint8,
                            device=p.device)
            if flags & 2:  # per-32 records: variant ss or block_n != 256
                _lib.call("itq3_repack_mmq_n", _lib.ptr(p), self.rows, self.cols, self.block_n,
                          int(self.variant == "ss"), int(not self.symmetric), _lib.ptr(t), _lib.stream_ptr(p.device))
            else:
                _lib.call("itq3_repack_mmq", _lib.ptr(p), self.rows, self.cols, flags, _lib.ptr(t),
                          _lib.stream_ptr(p.device))
            self._mmq[p.device] = t
        return self._mmq[p.device]

    def drop_payload(self) -> None:
        """Move the container-order payload to host memory once the tiled copy exists
        (GEMV-only serving keeps 66 B instead of 166 B per 256 weights on the device)."""
        if not self._tiled:
            raise ValueError("drop_payload: no tiled copy built")
        if self._payload is not None and self._payload.is_cuda:
            self._payload = self._payload.cpu()

    def device_nbytes(self) -> int:
        """Bytes this tensor holds on devices: the payload (if resident) plus every kernel layout built."""
        n = int(self._payload.numel()) if self._payload is not None and self._payload.is_cuda else 0
        for d in (self._tiled, self._mmq, self._mmq8):
            n += sum(int(t.numel()) for t in d.values())
        return n

    def release(self, *layouts: str) -> None:
        """Free device layouts this tensor no longer serves: "tiled" (GEMV / decode chain, 66 B per 256
        weights), "mmq" (K5, 70 B), "mmq8" (K5b, 67 B).  Each layout is rebuilt from the payload on next
        use, so a decode-only server keeps "tiled" (with `drop_payload`) and a prefill-only one "mmq"."""
        names = {"tiled": self._tiled, "mmq": self._mmq, "mmq8": self._mmq8}
        for name in layouts:
            if name not in names:
                raise ValueError(f"release: unknown layout {name!r}, expected one of {sorted(names)}")
            names[name].clear()
            if name == "tiled":
                self._chain1.clear()


# ------------------------------------------------------------------------------------------------
# validation (K7)
# ------------------------------------------------------------------------------------------------
def _raise_for(key: int, payload: torch.Tensor, n: int, ss: bool, prefix: bool) -> None:
    blk = key >> 16
    kind = (key >> 10) & 0x3F
    idx = key & 0x3FF
    raw = payload[blk].cpu().numpy().tobytes()
    b = block_from_bytes(raw, n, ss)
    if kind == 0:
        q = np.frombuffer(b.quants, np.uint8)
        bit = lambda p: (int(q[p * (n // 8) + (idx >> 3)]) >> (idx & 7)) & 1  # noqa: E731
        msg = f"unpack_ternary: stored code {bit(0) + 2 * bit(1) + 4 * bit(2)} > 2 at index {idx}"
    elif kind == 1:
        msg = "deserialize_block: scale is NaN"
    elif kind == 2:
        from .packing import decode_f16

        msg = f"deserialize_block: zero-point {decode_f16(b.zp_bits)} not in {{-1, 0, 1}}"
    elif kind == 3:
        msg = "deserialize_block: sub-scale is NaN"
    else:  # non-finite zero-point: PackedBlock.zp = int(decode_f16(bits)) raises in Python
        from .packing import decode_f16

        int(decode_f16(b.zp_bits))  # raises OverflowError / ValueError exactly like the reference
        msg = "zero-point is not finite"
    raise CorruptionError(f"block {blk}: {msg}" if prefix else msg)


def validate_payload(payload: torch.Tensor, n: int, ss: bool, full: bool, prefix: bool) -> None:
    """Run K7 over a device payload; raise the reference's error for the first offender."""
    mask = (_lib.CHECK_PLANES | _lib.CHECK_SCALE_NAN | _lib.CHECK_ZP | _lib.CHECK_SUB_NAN) if full else \
        (_lib.CHECK_PLANES | _lib.CHECK_ZP_FINITE)
    word = _lib.first_bad_word(payload.device)
    _lib.call("itq3_validate", _lib.ptr(payload), payload.shape[0], n, int(ss), mask, _lib.ptr(word),
              _lib.stream_ptr(payload.device))
    key = _lib.read_first_bad(word)
    if key is not None:
        _raise_for(key, payload, n, ss, prefix)


# ------------------------------------------------------------------------------------------------
# encode / decode
# ------------------------------------------------------------------------------------------------
def _weights_on_device(w, dev) -> torch.Tensor:
    if isinstance(w, torch.Tensor):
        t = w.detach()
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
        return t.to(dev).contiguous()
    a = np.asarray(w)
    if a.dtype != np.float32:
        a = np.asarray(a, dtype=np.float64)
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def _encode(t: torch.Tensor, cfg: QuantConfig) -> torch.Tensor:
    n = cfg.block_n
    ss = cfg.variant == "ss"
    nb = -(-t.numel() // n)
    payload = torch.empty((nb, block_nbytes(n, ss)), dtype=torch.uint8, device=t.device)
    dtype = _lib.F32 if t.dtype == torch.float32 else _lib.F64
    _lib.call("itq3_encode", _lib.ptr(t), dtype, t.numel(), n, int(ss), POLICY_CODE[cfg.policy.kind],
              cfg.policy.coefficient(), int(cfg.symmetric), _lib.ptr(payload), _lib.stream_ptr(t.device))
    return payload


def encode_block(w, cfg: QuantConfig) -> PackedBlock:
    """Rotate, quantize and pack one block (codec.py:113-149) with the K1 kernel."""
    a = np.asarray(w, dtype=np.float64) if not isinstance(w, torch.Tensor) else w
    if a.ndim != 1 or a.shape[0] != cfg.block_n:
        raise LengthError(f"encode_block: expected a 1-D block of length {cfg.block_n}, got shape {tuple(a.shape)}")
    dev = _lib.device()
    t = _weights_on_device(a, dev)
    if not bool(torch.isfinite(t).all()):
        raise DomainError("fwht_forward: input contains non-finite values")
    raw = _encode(t, cfg)[0].cpu().numpy().tobytes()
    return block_from_bytes(raw, cfg.block_n, cfg.variant == "ss")


def quantize_tensor(w, cfg: QuantConfig | None = None) -> QuantizedTensor:
    """Encode a 2-D matrix block by block in row-major order (codec.py:164-189)."""
    cfg = cfg or QuantConfig()
    shape = tuple(w.shape) if isinstance(w, torch.Tensor) else np.shape(w)
    if len(shape) != 2 or 0 in shape:
        raise ShapeError(f"quantize_tensor: expected a non-empty 2-D matrix, got shape {shape}")
    dev = _lib.device()
    t = _weights_on_device(w, dev)
    if not bool(torch.isfinite(t).all()):
        raise DomainError("quantize_tensor: input contains non-finite values")
    rows, cols = shape
    payload = _encode(t, cfg)
    pad = payload.shape[0] * cfg.block_n - rows * cols
    return QuantizedTensor(rows, cols, cfg.block_n, cfg.variant, cfg.symmetric, pad, payload=payload,
                           validated=True)


def _dequant_into(q: QuantizedTensor, out: torch.Tensor) -> torch.Tensor:
    p = q.ensure_decodable()
    code = {torch.float64: _lib.F64, torch.float32: _lib.F32}.get(out.dtype)
    if code is None or not out.is_contiguous() or out.numel() != q.rows * q.cols:
        raise ShapeError("dequantize_tensor: out must be a contiguous float32/float64 tensor of rows*cols")
    _lib.call("itq3_dequant", _lib.ptr(p), p.shape[0], q.block_n, int(q.variant == "ss"), q.rows * q.cols,
              _lib.ptr(out), code, _lib.stream_ptr(p.device))
    return out


def dequantize_tensor(q: QuantizedTensor, out: torch.Tensor | None = None):
    """Decode every block, strip the pad and reshape (codec.py:192-202).

    Returns a float64 numpy array (bit-identical to the reference); pass ``out=`` (a CUDA
    float32/float64 tensor) to decode straight into device memory instead.
    """
    if out is not None:
        return _dequant_into(q, out)
    dev = q.payload().device
    res = torch.empty((q.rows, q.cols), dtype=torch.float64, device=dev)
    return _dequant_into(q, res).cpu().numpy()


def decode_block(b: PackedBlock) -> np.ndarray:
    """Unpack, dequantize and inverse-rotate one block (codec.py:152-161)."""
    q = QuantizedTensor(1, b.n, b.n, "ss" if b.sub_scale_bits is not None else "s", True, 0, blocks=[b])
    p = q.payload()
    validate_payload(p, b.n, b.sub_scale_bits is not None, full=False, prefix=False)
    q._validated = True
    return dequantize_tensor(q)[0]


# ------------------------------------------------------------------------------------------------
# container (codec.py:205-291)
# ------------------------------------------------------------------------------------------------
def _check_tensor(q: QuantizedTensor) -> None:
    if q.variant not in VARIANTS:
        raise DomainError(f"container: unknown variant {q.variant!r}")
    if q.block_n not in BLOCK_SIZES:
        raise DomainError(f"container: invalid block_n {q.block_n}")
    if not (0 <= q.pad < q.block_n):
        raise DomainError(f"container: pad {q.pad} out of range for block_n {q.block_n}")
    if len(q) != q.n_blocks:
        raise ShapeError(f"container: {len(q)} blocks, expected {q.n_blocks}")


def write_container(q: QuantizedTensor, sink) -> int:
    """Header + payload bytes (device -> host copy of the resident payload)."""
    _check_tensor(q)
    flags = (FLAG_SUB_SCALES if q.variant == "ss" else 0) | (0 if q.symmetric else FLAG_ASYMMETRIC)
    header = HEADER.pack(MAGIC, VERSION, flags, q.rows, q.cols, q.block_n, q.pad)
    body = q.payload().cpu().numpy().tobytes()
    if hasattr(sink, "write"):
        sink.write(header)
        sink.write(body)
    else:
        with open(sink, "wb") as f:
            f.write(header)
            f.write(body)
    return len(header) + len(body)


_STAGE_BYTES = 64 << 20  # pinned staging chunk for container ingest


class _Staging:
    """Two reusable pinned host chunks: chunk i+1 is filled from the file while chunk i's H2D copy runs."""

    def __init__(self):
        self.bufs = []
        self.events = []

    def get(self, i: int, dev) -> tuple[torch.Tensor, torch.cuda.Event]:
        while len(self.bufs) < 2:
            self.bufs.append(torch.empty(_STAGE_BYTES, dtype=torch.uint8, pin_memory=True))
            self.events.append(torch.cuda.Event())
        ev = self.events[i % 2]
        ev.synchronize()  # the previous copy out of this chunk has finished
        return self.bufs[i % 2], ev


_staging = _Staging()


def _ingest(reader, nbytes: int, dev) -> torch.Tensor:
    """Stream nbytes from reader(memoryview) -> count into a device tensor through pinned chunks."""
    out = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    off, i = 0, 0
    while off < nbytes:
        buf, ev = _staging.get(i, dev)
        take = min(buf.numel(), nbytes - off)
        view = memoryview(buf.numpy())[:take]
        got = 0
        while got < take:
            k = reader(view[got:])
            if not k:
                break
            got += k
        if got < take:
            return out[:off + got]  # short read: caller reports truncation
        out[off:off + take].copy_(buf[:take], non_blocking=True)
        ev.record(stream)
        off += take
        i += 1
    return out


def read_container(source) -> QuantizedTensor:
    """Parse the header on the host, stream the payload to the GPU through pinned staging
    (file reads overlap the H2D copies), and validate every block with one K7 pass."""
    close = None
    if hasattr(source, "read") and not (hasattr(source, "seekable") and source.seekable()):
        source = source.read()  # pipes / unseekable streams: the length is only known at EOF
    if isinstance(source, (bytes, bytearray, memoryview)):
        mv = memoryview(source).cast("B")
        pos = [0]

        def reader(dst):
            k = min(len(dst), len(mv) - pos[0])
            dst[:k] = mv[pos[0]:pos[0] + k]
            pos[0] += k
            return k

        remaining = lambda: len(mv) - pos[0]  # noqa: E731
    else:
        f = source if hasattr(source, "read") else open(source, "rb")
        close = None if f is source else f
        if hasattr(f, "readinto"):
            reader = f.readinto
        else:
            def reader(dst):
                b = f.read(len(dst))
                dst[:len(b)] = b
                return len(b)

        def remaining():
            try:
                return os.fstat(f.fileno()).st_size - f.tell()
            except (AttributeError, OSError, io.UnsupportedOperation):
                here = f.tell()
                end = f.seek(0, io.SEEK_END)
                f.seek(here)
                return end - here
    try:
        head = bytearray(HEADER.size)
        got = 0
        while got < HEADER.size:
            k = reader(memoryview(head)[got:])
            if not k:
                break
            got += k
        if got < HEADER.size:
            raise TruncatedStreamError(f"container header needs {HEADER.size} bytes, got {got}")
        magic, version, flags, rows, cols, block_n, pad = HEADER.unpack_from(head, 0)
        if magic != MAGIC:
            raise BadMagicError(f"bad magic {magic!r}, expected {MAGIC!r}")
        if version != VERSION:
            raise UnsupportedVersionError(f"unsupported container version {version}")
        if flags & ~KNOWN_FLAGS:
            raise ContainerError(f"unknown flag bits 0x{flags & ~KNOWN_FLAGS:x}")
        if block_n not in BLOCK_SIZES:
            raise ContainerError(f"invalid block_n {block_n}")
        if rows == 0 or cols == 0:
            raise ContainerError(f"empty tensor dims {rows}x{cols}")
        n_blocks = -(-rows * cols // block_n)
        if pad != n_blocks * block_n - rows * cols:
            raise ContainerError(f"pad {pad} inconsistent with {rows}x{cols} at block_n {block_n}")
        ss = bool(flags & FLAG_SUB_SCALES)
        bsize = block_nbytes(block_n, ss)
        expected = HEADER.size + n_blocks * bsize
        have = HEADER.size + remaining()
        if have < expected:
            raise TruncatedStreamError(f"container truncated: expected {expected} bytes, got {have}")
        if have > expected:
            raise SizeMismatchError(f"container has {have - expected} trailing bytes (expected {expected}, got {have})")
        dev = _lib.device()
        flat = _ingest(reader, n_blocks * bsize, dev)
        if flat.numel() < n_blocks * bsize:
            raise TruncatedStreamError(f"container truncated: expected {expected} bytes, "
                                       f"got {HEADER.size + flat.numel()}")
    finally:
        if close is not None:
            close.close()
    payload = flat.view(n_blocks, bsize)
    validate_payload(payload, block_n, ss, full=True, prefix=True)
    return QuantizedTensor(rows, cols, block_n, "ss" if ss else "s", not (flags & FLAG_ASYMMETRIC), pad,
                           payload=payload, validated=True)
