"""Container ingest: read_container streams the payload through pinned staging
chunks to the GPU and validates it with one K7 pass.  Checked against the reference's golden
containers from every source kind, across chunk boundaries, and for truncation/trailing bytes."""

import io
import os

import numpy as np
import pytest

import paper_2603_27914_b200 as P
import paper_2603_27914_b200.codec as C

pytestmark = pytest.mark.gpu


class Unseekable(io.RawIOBase):
    def __init__(self, data):
        self.b = io.BytesIO(data)

    def readable(self):
        return True

    def seekable(self):
        return False

    def readinto(self, buf):
        return self.b.readinto(buf)


@pytest.mark.parametrize("stage", [C._STAGE_BYTES, 4096, 1000])
def test_ingest_all_sources_and_chunkings(golden, tmp_path, monkeypatch, stage):
    monkeypatch.setattr(C, "_STAGE_BYTES", stage)
    monkeypatch.setattr(C, "_staging", C._Staging())
    meta, arrays, _ = golden
    for c in meta[::11]:
        data = arrays[c["key"] + "_container"].tobytes()
        path = tmp_path / "c.itq3"
        path.write_bytes(data)
        ref = P.read_container(data)
        for src in (bytearray(data), memoryview(data), io.BytesIO(data), str(path), path, Unseekable(data)):
            q = P.read_container(src)
            assert q == ref
            buf = io.BytesIO()
            P.write_container(q, buf)
            assert buf.getvalue() == data
        with open(path, "rb") as f:  # reads from the current position of an open file
            assert P.read_container(f) == ref


def test_ingest_errors(golden, tmp_path):
    meta, arrays, _ = golden
    data = arrays[meta[0]["key"] + "_container"].tobytes()
    p = tmp_path / "t.itq3"
    p.write_bytes(data[:-7])
    with pytest.raises(P.TruncatedStreamError, match="truncated"):
        P.read_container(str(p))
    p.write_bytes(data + b"\0")
    with pytest.raises(P.SizeMismatchError, match="1 trailing bytes"):
        P.read_container(str(p))
    with pytest.raises(P.TruncatedStreamError, match="header needs 32 bytes, got 5"):
        P.read_container(io.BytesIO(data[:5]))
    bad = bytearray(data)
    n = meta[0]["block_n"]
    bad[32] |= 0x01  # element 0: plane 0 ...
    bad[32 + n // 8] |= 0x01  # ... and plane 1 -> stored code 3
    with pytest.raises(P.CorruptionError, match="block 0"):
        P.read_container(Unseekable(bytes(bad)))


def test_ingest_large_multichunk():
    rng = np.random.default_rng(0)
    w = rng.standard_normal((1536, 4096)).astype(np.float32)
    q = P.quantize_tensor(w)
    buf = io.BytesIO()
    n = P.write_container(q, buf)
    assert n == 32 + 1536 * 16 * 100
    old = C._STAGE_BYTES
    try:
        C._STAGE_BYTES = 1 << 20
        C._staging = C._Staging()
        q2 = P.read_container(buf.getvalue())
    finally:
        C._STAGE_BYTES = old
        C._staging = C._Staging()
    assert q2 == q
