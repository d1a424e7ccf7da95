"""SPRM remap files: byte compatibility with the reference's
write_remap / read_remap (core/src/remap.cpp:118-176) and its error behaviour.

Host-location calls are pure file I/O through the C-ABI (no GPU); the device
round trip streams through pinned memory and counts slow rows on the GPU.
"""
import os
import struct

import numpy as np
import pytest

import oracle
import paper_2201_10095_b200 as sp
from paper_2201_10095_b200.types import IoError, ParseError, RemapTable

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def _table(H=1000, hbm=300, seed=0, table_id=7):
    rng = np.random.default_rng(seed)
    ent = np.empty(H, np.int32)
    perm = rng.permutation(H)
    ent[perm[:hbm]] = np.arange(hbm, dtype=np.int32)
    ent[perm[hbm:]] = -1 - np.arange(H - hbm, dtype=np.int32)
    return RemapTable(table_id, H, hbm, H - hbm, ent)


@needs_ref
@pytest.mark.parametrize("H,hbm", [(0, 0), (1, 0), (1, 1), (1000, 300), (4097, 4097)])
def test_write_is_byte_identical_to_reference(tmp_path, H, hbm):
    r = _table(H, hbm, seed=H)
    ours, theirs = tmp_path / "ours.sprm", tmp_path / "ref.sprm"
    sp.write_remap(r, ours)
    oracle.Ref().write_remap(theirs, r.table_id, r.hash_size, r.hbm_rows, r.entries)
    assert ours.read_bytes() == theirs.read_bytes()
    assert len(ours.read_bytes()) == r.serialized_bytes()


@needs_ref
def test_read_reference_written_file(tmp_path):
    r = _table(5000, 1234, seed=3, table_id=0xFFFFFFFF)
    p = tmp_path / "ref.sprm"
    oracle.Ref().write_remap(p, r.table_id, r.hash_size, r.hbm_rows, r.entries)
    got = sp.read_remap(p)
    want = oracle.Ref().read_remap(p)
    assert (got.table_id, got.hash_size, got.hbm_rows, got.slow_rows_allocated) == (
        want["table_id"], want["hash_size"], want["hbm_rows"], want["slow_rows_allocated"])
    assert np.array_equal(got.entries, want["entries"])
    assert got.slow_rows_allocated == 5000 - 1234


def test_header_layout(tmp_path):
    """29-byte header: "SPRM", version 1, table_id/hash_size/hbm_rows as u64 LE."""
    r = _table(3, 2, table_id=5)
    p = tmp_path / "t.sprm"
    sp.write_remap(r, p)
    b = p.read_bytes()
    assert b[:5] == b"SPRM\x01"
    assert struct.unpack("<QQQ", b[5:29]) == (5, 3, 2)
    assert np.array_equal(np.frombuffer(b[29:], "<i4"), r.entries)


def _expect(exc, msg, path):
    with pytest.raises(exc) as e:
        sp.read_remap(path)
    assert msg + str(path) in str(e.value)
    if oracle.ref_available():
        with pytest.raises(oracle.OracleError) as e2:
            oracle.Ref().read_remap(path)
        assert e2.value.status == {IoError: -4, ParseError: -2}[exc]
        assert msg + str(path) in str(e2.value)


def test_read_errors_match_reference(tmp_path):
    _expect(IoError, "cannot open: ", tmp_path / "missing.sprm")
    short = tmp_path / "short.sprm"
    short.write_bytes(b"SPRM\x01" + b"\0" * 10)
    _expect(ParseError, "remap file too short: ", short)
    bad = tmp_path / "bad.sprm"
    bad.write_bytes(b"SPRX\x01" + struct.pack("<QQQ", 0, 0, 0))
    _expect(ParseError, "bad remap magic or version: ", bad)
    ver = tmp_path / "ver.sprm"
    ver.write_bytes(b"SPRM\x02" + struct.pack("<QQQ", 0, 0, 0))
    _expect(ParseError, "bad remap magic or version: ", ver)
    big = tmp_path / "big.sprm"
    big.write_bytes(b"SPRM\x01" + struct.pack("<QQQ", 0, 1 << 31, 0))
    _expect(ParseError, "remap hash_size out of range: ", big)
    trunc = tmp_path / "trunc.sprm"
    trunc.write_bytes(b"SPRM\x01" + struct.pack("<QQQ", 0, 10, 0) + b"\0" * 36)
    _expect(ParseError, "remap file truncated: ", trunc)


def test_write_errors(tmp_path):
    with pytest.raises(IoError, match="cannot open for writing: "):
        sp.write_remap(_table(4, 1), tmp_path / "no_such_dir" / "x.sprm")
    r = _table(4, 1)
    r.entries = r.entries[:3]
    with pytest.raises(sp.InvalidArgument):
        sp.write_remap(r, tmp_path / "x.sprm")


@pytest.mark.gpu
@pytest.mark.parametrize("H", [1, 1000, (8 << 20) * 2 + 12345])
def test_device_round_trip(cuda_ctx, tmp_path, H):
    """Device entries -> file -> device, chunked through pinned memory both ways
    (the largest case crosses the 8M-entry read double buffer twice)."""
    import torch

    r = _table(H, H // 3, seed=H)
    p_host, p_dev = tmp_path / "h.sprm", tmp_path / "d.sprm"
    sp.write_remap(r, p_host)
    rd = RemapTable(r.table_id, H, r.hbm_rows, r.slow_rows_allocated,
                    torch.from_numpy(r.entries).cuda())
    sp.write_remap(rd, p_dev)
    assert p_host.read_bytes() == p_dev.read_bytes()
    got = sp.read_remap(p_host, device=True)
    assert got.entries.is_cuda and got.entries.dtype == torch.int32
    assert np.array_equal(got.entries.cpu().numpy(), r.entries)
    assert got.slow_rows_allocated == H - H // 3
    assert (got.table_id, got.hash_size, got.hbm_rows) == (r.table_id, H, H // 3)


@pytest.mark.gpu
def test_device_read_truncated(cuda_ctx, tmp_path):
    trunc = tmp_path / "trunc.sprm"
    trunc.write_bytes(b"SPRM\x01" + struct.pack("<QQQ", 0, 10, 0) + b"\0" * 36)
    with pytest.raises(ParseError, match="remap file truncated: "):
        sp.read_remap(trunc, device=True)
