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


# ----------------------------------------------------------------------------- sz3g_stream_validate
def _book(pairs):
    import struct
    return struct.pack("<I", len(pairs)) + b"".join(struct.pack("<HB", s, l) for s, l in pairs)


def _valid(n_out=2, dim0_offset=12, lr=False):
    """A consistent compressed-field stream for dims (2, 3, 4) (N = 24, one block, one chunk)."""
    import struct
    plane = 3 * 4
    idx = [dim0_offset * plane + 5, dim0_offset * plane + 23][:n_out]
    secs = [
        (sz3g.SEC_CODE_BOOK, _book([(32767, 1), (32768, 1)])),
        (sz3g.SEC_CODE_OFFS, struct.pack("<QQ", 0, 1)),
        (sz3g.SEC_CODE_DATA, b"\x00" * 4),
        (sz3g.SEC_COEF_BOOK, _book([(0, 1), (7, 1)])),
        (sz3g.SEC_COEF_OFFS, struct.pack("<QQ", 0, 1)),
        (sz3g.SEC_COEF_DATA, b"\x00" * 4),
        (sz3g.SEC_COEF_ESC, b""),
        (sz3g.SEC_OUT_IDX, struct.pack(f"<{n_out}Q", *idx)),
        (sz3g.SEC_OUT_VAL, struct.pack(f"<{n_out}f", *([1.5] * n_out))),
    ]
    if lr:
        secs.append((sz3g.SEC_LR_FLAGS, b"\x01"))
    hdr = sz3g.StreamHeader(0, 3, (ctypes.c_uint64 * 3)(2, 3, 4), 1, 1e-3, 0.5, 32768, 6, 2048, 16,
                            sz3g.STREAM_LR if lr else 0, n_out, 1, dim0_offset)
    return hdr, secs


def validate(hdr, secs):
    lib = sz3g.load()
    arr = (sz3g.Section * max(1, len(secs)))()
    keep = []
    for i, (tag, b) in enumerate(secs):
        buf = ctypes.create_string_buffer(b, len(b)) if b else None
        keep.append(buf)
        arr[i] = sz3g.Section(tag, ctypes.cast(buf, ctypes.c_void_p) if buf else None, len(b))
    bad = ctypes.c_uint32(99)
    rc = lib.sz3g_stream_validate(ctypes.byref(hdr), arr, len(secs), ctypes.byref(bad))
    return rc, bad.value


def test_validate_accepts_consistent_stream_and_keeps_dim0_offset():
    hdr, secs = _valid()
    assert validate(hdr, secs) == (0, 0)
    assert validate(*_valid(lr=True)) == (0, 0)
    # dim0_offset survives the container (outlier indices are global)
    rc, h2, got, _ = read(pack(secs, hdr))
    assert rc == 0 and h2.dim0_offset == 12 and validate(h2, got) == (0, 0)


def _mut(fn):
    hdr, secs = _valid()
    secs = [list(s) for s in secs]
    fn(hdr, secs)
    return validate(hdr, [tuple(s) for s in secs])


@pytest.mark.parametrize("case,tag", [
    ("n_outliers_too_big", 8), ("nblocks", 0), ("ndim0", 0), ("radius", 0), ("eb_abs_nan", 0),
    ("outlier_outside_slab", 8), ("offsets_not_monotone", 2), ("offsets_past_payload", 2),
    ("offsets_count", 2), ("book_symbol_range", 1), ("book_len_zero", 4), ("missing_section", 6),
    ("lr_flag_without_section", 10), ("out_val_size", 9), ("leading_extent", 0)])
def test_validate_rejects_inconsistent_stream(case, tag):
    import struct

    def f(h, s):
        if case == "n_outliers_too_big":
            h.n_outliers = 3
        elif case == "nblocks":
            h.nblocks = 2
        elif case == "ndim0":
            h.ndim = 0
        elif case == "radius":
            h.radius = 40000
        elif case == "eb_abs_nan":
            h.eb_abs = float("nan")
        elif case == "outlier_outside_slab":
            s[7][1] = struct.pack("<2Q", 12 * 12 + 5, 12 * 12 + 24)   # one past the slab end
        elif case == "offsets_not_monotone":
            s[1][1] = struct.pack("<QQ", 1, 0)
        elif case == "offsets_past_payload":
            s[1][1] = struct.pack("<QQ", 0, 2)
        elif case == "offsets_count":
            s[1][1] = struct.pack("<QQQ", 0, 1, 1)
        elif case == "book_symbol_range":
            h.radius = 100            # the code book's symbols 32767, 32768 are >= 2R
        elif case == "book_len_zero":
            s[3][1] = _book([(3, 0)])
        elif case == "missing_section":
            del s[5]
        elif case == "lr_flag_without_section":
            h.flags = sz3g.STREAM_LR
        elif case == "out_val_size":
            s[8][1] = s[8][1][:4]
        elif case == "leading_extent":
            h.ndim = 2
    rc, bad = _mut(f)
    assert rc == -5 and bad == tag, (case, rc, bad)


def _valid_interp():
    """A consistent SZ3-Interp stream: no coefficient sections, nblocks 0."""
    hdr, secs = _valid()
    secs = [s for s in secs if s[0] not in (sz3g.SEC_COEF_BOOK, sz3g.SEC_COEF_OFFS, sz3g.SEC_COEF_DATA,
                                             sz3g.SEC_COEF_ESC)]
    hdr.flags = sz3g.STREAM_INTERP
    hdr.nblocks = 0
    return hdr, secs


def test_validate_interp_streams():
    assert validate(*_valid_interp()) == (0, 0)
    hdr, secs = _valid_interp()
    hdr.nblocks = 1                                    # an Interp stream carries no blocks
    assert validate(hdr, secs)[0] == -5
    hdr, secs = _valid_interp()
    hdr.flags = sz3g.STREAM_INTERP | sz3g.STREAM_LR    # exclusive
    assert validate(hdr, secs)[0] == -5
    hdr, secs = _valid()
    hdr.flags = sz3g.STREAM_INTERP                     # coefficient sections present
    hdr.nblocks = 0
    rc, bad = validate(hdr, secs)
    assert rc == -5 and bad == sz3g.SEC_COEF_BOOK
    hdr, secs = _valid()
    hdr.flags = 0x8                                    # unknown flag
    assert validate(hdr, secs)[0] == -5
