"""CBV1 container (the BV stream on disk), tested the
way the reference specifies its RMV1 container (rmv_io.hpp:31-49):
deterministic bytes, exact round trip, FormatError for an unrecognised
container, CorruptionError for truncation, trailing bytes and damaged
contents, and no partial results.  CPU only."""
import os
import struct

import numpy as np
import pytest

import paper_1708_07271_b200 as P
from tests.helpers import csr_from_rows


def _stream(n=3000, deg=12.0, seed=3, **kw):
    g = P.CsrGraph.copy_model(n, deg, seed=seed)
    return g, P.BvStream.encode(g, P.BvParams(**kw))


def test_roundtrip_bytes_and_file(tmp_path):
    g, s = _stream()
    b = s.to_bytes()
    assert b[:4] == b"CBV1" and b[4] == 1
    assert s.to_bytes() == b  # deterministic
    t = P.BvStream.from_bytes(b)
    assert (t.n, t.m, t.params) == (s.n, s.m, s.params)
    assert np.array_equal(t.words()[: (s.stats()["stream_bits"] + 31) // 32],
                          s.words()[: (s.stats()["stream_bits"] + 31) // 32])
    assert np.array_equal(t.segment_offsets(), s.segment_offsets())
    assert t.to_bytes() == b  # re-encoding the loaded stream gives the same bytes
    d = t.decode_host()
    assert np.array_equal(d.row_offsets, g.row_offsets) and np.array_equal(d.columns, g.columns)
    st, ss = t.stats(), s.stats()
    assert st["stream_bits"] == ss["stream_bits"] and st["rows_with_ref"] == ss["rows_with_ref"]
    assert st["max_depth"] == ss["max_depth"]
    p = tmp_path / "g.cbv"
    s.save(str(p))
    assert p.read_bytes() == b
    u = P.BvStream.load(str(p))
    assert u.to_bytes() == b


@pytest.mark.parametrize("kw", [dict(max_ref=0), dict(window=3, min_interval=2), dict(segment_rows=256)])
def test_roundtrip_params(kw):
    g, s = _stream(n=2500, **kw)
    t = P.BvStream.from_bytes(s.to_bytes())
    assert t.params == s.params
    d = t.decode_host()
    assert np.array_equal(d.columns, g.columns)


def test_edge_cases_empty_rows_and_empty_graph():
    g = csr_from_rows([[], [0], [], [0, 1, 2], []])
    s = P.BvStream.encode(g, P.BvParams())
    t = P.BvStream.from_bytes(s.to_bytes())
    assert np.array_equal(t.decode_host().columns, g.columns)
    g0 = csr_from_rows([[] for _ in range(4)])
    s0 = P.BvStream.encode(g0, P.BvParams())
    assert P.BvStream.from_bytes(s0.to_bytes()).m == 0


def test_format_errors():
    _, s = _stream(n=500)
    b = bytearray(s.to_bytes())
    with pytest.raises(P.FormatError):
        P.BvStream.from_bytes(b"RMV1" + bytes(b[4:]))
    with pytest.raises(P.FormatError):
        P.BvStream.from_bytes(bytes(b[:4]) + b"\x02" + bytes(b[5:]))
    with pytest.raises(P.FormatError):
        P.BvStream.from_bytes(b"")


def test_corruption_errors():
    _, s = _stream(n=500)
    b = s.to_bytes()
    with pytest.raises(P.CorruptionError):  # truncated header
        P.BvStream.from_bytes(b[:20])
    with pytest.raises(P.CorruptionError):  # truncated body
        P.BvStream.from_bytes(b[:-9])
    with pytest.raises(P.CorruptionError):  # trailing bytes
        P.BvStream.from_bytes(b + b"\x00")
    rng = np.random.default_rng(0)
    for pos in rng.integers(8, len(b) - 8, size=20):  # any flipped bit in the body: checksum
        bad = bytearray(b)
        bad[pos] ^= 1 << int(rng.integers(0, 8))
        with pytest.raises((P.CorruptionError, P.FormatError)):
            P.BvStream.from_bytes(bytes(bad))


def test_corrupt_contents_with_valid_checksum():
    """A container whose checksum matches but whose contents violate an
    invariant (edge count, segment table) is still rejected."""
    _, s = _stream(n=500)
    b = bytearray(s.to_bytes())

    def reseal(buf):
        h = 0xcbf29ce484222325
        for c in bytes(buf[:-8]):
            h = ((h ^ c) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
        buf[-8:] = struct.pack("<Q", h)
        return bytes(buf)

    bad = bytearray(b)
    m = struct.unpack_from("<Q", bad, 12)[0]
    struct.pack_into("<Q", bad, 12, m + 1)  # header m
    with pytest.raises(P.CorruptionError):
        P.BvStream.from_bytes(reseal(bad))
    bad = bytearray(b)
    struct.pack_into("<I", bad, 36, 0)  # segment_rows = 0
    with pytest.raises(P.CorruptionError):
        P.BvStream.from_bytes(reseal(bad))
    bad = bytearray(b)
    struct.pack_into("<Q", bad, 60, 1)  # first segment offset != 0
    with pytest.raises(P.CorruptionError):
        P.BvStream.from_bytes(reseal(bad))


def test_load_missing_file(tmp_path):
    with pytest.raises(ValueError):  # invalid_argument, as for an unusable path
        P.BvStream.load(str(tmp_path / "missing.cbv"))


def test_loaded_stream_keeps_edge_statistics():
    """A loaded container recomputes the encoder's edge statistics from the
    decoded rows (cmv::stats on a loaded stream, ref_matrix.hpp:78-89)."""
    g = P.CsrGraph.copy_model(6000, 10.0, seed=3)
    s = P.BvStream.encode(g, P.BvParams())
    assert P.BvStream.from_bytes(s.to_bytes()).stats() == s.stats()
