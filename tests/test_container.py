"""The self-describing stream container (sz3g_stream_*): host C++ in libsz3g, testable on
the CPU.  Round trip of header and sections; every corruption is rejected -- bad magic, bad version, a
flipped payload byte (reported with its section tag), a truncated stream, trailing bytes."""
from __future__ import annotations

import ctypes

import pytest

from paper_2111_02925_b200 import sz3g


def pack(sections, hdr=None):
    lib = sz3g.load()
    hdr = hdr or sz3g.StreamHeader(0, 3, (ctypes.c_uint64 * 3)(2, 3, 4), 1, 1e-3, 0.5, 32768, 6, 2048, 16, 0, 7, 9)
    secs = (sz3g.Section * len(sections))()
    keep = []
    for i, (tag, b) in enumerate(sections):
        buf = ctypes.create_string_buffer(b, len(b)) if b else None
        keep.append(buf)
        secs[i] = sz3g.Section(tag, ctypes.cast(buf, ctypes.c_void_p) if buf else None, len(b))
    size = lib.sz3g_stream_size(secs, len(sections))
    out = ctypes.create_string_buffer(size)
    wr = ctypes.c_uint64(0)
    assert lib.sz3g_stream_write(ctypes.byref(hdr), secs, len(sections), out, size, ctypes.byref(wr)) == 0
    assert wr.value == size
    return out.raw


def read(b):
    lib = sz3g.load()
    hdr = sz3g.StreamHeader()
    secs = (sz3g.Section * 16)()
    n, bad = ctypes.c_uint32(0), ctypes.c_uint32(0)
    rc = lib.sz3g_stream_read(b, len(b), ctypes.byref(hdr), secs, 16, ctypes.byref(n), ctypes.byref(bad))
    got = [(secs[i].tag, ctypes.string_at(secs[i].data, secs[i].bytes)) for i in range(n.value)] if rc == 0 else None
    return rc, hdr, got, bad.value


SECTIONS = [(1, b"\x02\x00\x00\x00abcdef"), (3, bytes(range(256)) * 3), (7, b""), (9, b"\xff" * 13)]


def test_round_trip():
    b = pack(SECTIONS)
    assert b[:4] == b"SZ3G"
    rc, hdr, got, _ = read(b)
    assert rc == 0 and got == SECTIONS
    assert tuple(hdr.dims) == (2, 3, 4) and hdr.eb == 1e-3 and hdr.eb_abs == 0.5 and hdr.radius == 32768
    assert hdr.chunk == 2048 and hdr.max_len == 16 and hdr.n_outliers == 7 and hdr.nblocks == 9


@pytest.mark.parametrize("where,tag", [(-1, 9), (-20, 9), (200, 3)])
def test_flipped_payload_byte_names_the_section(where, tag):
    b = bytearray(pack(SECTIONS))
    if where > 0:   # inside section 3's payload: after magic, version, header, nsec, section 1
        where = 4 + 2 + 96 + 4 + (1 + 8 + 8 + 10) + (1 + 8 + 8) + 50
    b[where] ^= 0x40
    rc, _, _, bad = read(bytes(b))
    assert rc == -5 and bad == tag


def test_bad_magic_version_truncation_trailing():
    b = pack(SECTIONS)
    assert read(b"SZ3X" + b[4:])[0] == -5
    assert read(b[:4] + b"\x02\x00" + b[6:])[0] == -5
    assert read(b[:-1])[0] == -5
    assert read(b + b"\x00")[0] == -5
    assert read(b[:50])[0] == -5
