"""NC06 hybrid binary format ("Hybrid Binary Compression (NC06)"; P:571-572;
S:377-499).  CPU ORACLE -- test infrastructure only (see oracle/__init__.py).

Segmentation, rules applied once each, in the paper's order, with adjacent
same-kind regions merged after every rule (reading D33):
  (1) bytes in printable ASCII 32..126 plus tab / LF / CR are text-like, runs of them are
      text regions, everything else binary;
  (2) text runs shorter than 64 bytes are demoted to binary;
  (3) binary gaps of <= 8 bytes between two text runs are bridged (relabelled text);
  (4) binary chunks shorter than 64 bytes adjacent to text are absorbed (relabelled text).
Bytes are never altered, only labelled.

Binary blob: every binary region concatenated in order, compressed with LZMA
(.xz stream, preset 6, CRC64) when the blob is >= 4 KB, else with DEFLATE (zlib stream,
level 9; the paper's "gzip", reading D34), stored raw if the codec output is not strictly
smaller; method byte 0 raw, 1 DEFLATE, 2 LZMA.  The codecs are library
routines (Python's lzma / zlib).

Text: the text regions concatenated into one document, chunked and
compressed by the NC05 text pipeline (oracle/compressor.py).

Container (little-endian; the field layout is SPEC's, reading D34):
  b"NC06" | version u8 = 1 | flags u8 | tau_milli u16 | entry_count u16
  | entry_count x {kind u8 (0 binary, 1 text), original_length u32}
  | method u8 | blob_length u32 | blob
  | chunk_count u16 | chunk_count x {token_count u32, bit_count u32, stream_len u32} | streams
An input with more than 65,535 regions is stored as a single binary entry (reading D34).
"""
import lzma
import struct
import zlib

from .container import FormatError

TEXT, BINARY = 1, 0
MIN_TEXT = 64        # rule 2: "short text runs (<64 bytes) are demoted"
MAX_GAP = 8          # rule 3: "binary gaps <= 8 bytes ... are bridged"
MIN_BIN = 64         # rule 4: "small binary chunks (<64 bytes) adjacent to text are absorbed"
LZMA_MIN = 4096      # "LZMA (>= 4 KB blobs) or gzip (smaller)"
RAW, DEFLATE, LZMA = 0, 1, 2


def is_text_byte(b: int) -> bool:
    """rule 1: printable ASCII (32-126) plus tab / LF / CR."""
    return 32 <= b <= 126 or b in (9, 10, 13)


def _merge(regs):
    out = []
    for k, ln in regs:
        if ln == 0:
            continue
        if out and out[-1][0] == k:
            out[-1] = (k, out[-1][1] + ln)
        else:
            out.append((k, ln))
    return out


def segment(data: bytes):
    """[(kind, length)] covering data in order (kinds alternate)."""
    regs = []
    for b in data:                                      # rule 1: runs of the byte class
        k = TEXT if is_text_byte(b) else BINARY
        if regs and regs[-1][0] == k:
            regs[-1][1] += 1
        else:
            regs.append([k, 1])
    regs = _merge([tuple(r) for r in regs])
    # rule 2: demote short text runs
    regs = _merge([(BINARY if k == TEXT and ln < MIN_TEXT else k, ln) for k, ln in regs])
    # rule 3: bridge short binary gaps between text runs
    regs = _merge([(TEXT if (k == BINARY and ln <= MAX_GAP and 0 < i < len(regs) - 1
                             and regs[i - 1][0] == TEXT and regs[i + 1][0] == TEXT) else k, ln)
                   for i, (k, ln) in enumerate(regs)])
    # rule 4: absorb small binary chunks adjacent to text
    regs = _merge([(TEXT if (k == BINARY and ln < MIN_BIN and
                             ((i > 0 and regs[i - 1][0] == TEXT) or (i + 1 < len(regs) and regs[i + 1][0] == TEXT)))
                    else k, ln) for i, (k, ln) in enumerate(regs)])
    return regs


def blob_encode(blob: bytes):
    """(method, payload): LZMA if >= 4 KB else DEFLATE, raw unless strictly smaller."""
    if not blob:
        return RAW, b""
    if len(blob) >= LZMA_MIN:
        m, c = LZMA, lzma.compress(blob, format=lzma.FORMAT_XZ, check=lzma.CHECK_CRC64, preset=6)
    else:
        m, c = DEFLATE, zlib.compress(blob, 9)
    return (m, c) if len(c) < len(blob) else (RAW, blob)


def blob_decode(method: int, payload: bytes) -> bytes:
    if method == RAW:
        return payload
    if method == DEFLATE:
        return zlib.decompress(payload)
    if method == LZMA:
        return lzma.decompress(payload, format=lzma.FORMAT_XZ)
    raise FormatError("unknown blob method")


def split(data: bytes, regs):
    """(text document, binary blob) from a segmentation."""
    text, binary, off = [], [], 0
    for k, ln in regs:
        (text if k == TEXT else binary).append(data[off:off + ln])
        off += ln
    return b"".join(text), b"".join(binary)


def write_nc06(flags, tau_milli, regs, method, payload, chunks):
    """chunks: NC05-style [(token_count, bit_count, stream)] of the text document."""
    if len(regs) > 0xFFFF or len(chunks) > 0xFFFF:
        raise FormatError("too many entries / chunks")
    out = [b"NC06", struct.pack("<BBHH", 1, flags, tau_milli, len(regs))]
    out += [struct.pack("<BI", k, ln) for k, ln in regs]
    out.append(struct.pack("<BI", method, len(payload)))
    out.append(payload)
    out.append(struct.pack("<H", len(chunks)))
    for n, bits, s in chunks:
        if len(s) != (bits + 7) // 8:
            raise FormatError("stream_len != ceil(bit_count/8)")
        out.append(struct.pack("<III", n, bits, len(s)))
    out += [s for _, _, s in chunks]
    return b"".join(out)


def read_nc06(data: bytes):
    """-> (flags, tau_milli, regs, method, payload, chunks)."""
    if len(data) < 10:
        raise FormatError("truncated header")
    if data[:4] != b"NC06":
        raise FormatError("bad magic")
    ver, flags, tau_milli, ne = struct.unpack_from("<BBHH", data, 4)
    if ver != 1:
        raise FormatError("unsupported NC06 version")
    if flags & ~0x07:
        raise FormatError("reserved flag bits set")
    off = 10
    if len(data) < off + 5 * ne + 5:
        raise FormatError("truncated entry table")
    regs = [struct.unpack_from("<BI", data, off + 5 * i) for i in range(ne)]
    if any(k not in (TEXT, BINARY) for k, _ in regs):
        raise FormatError("bad entry kind")
    off += 5 * ne
    method, bl = struct.unpack_from("<BI", data, off)
    off += 5
    if off + bl + 2 > len(data):
        raise FormatError("truncated binary section")
    payload = bytes(data[off:off + bl])
    off += bl
    (nch,) = struct.unpack_from("<H", data, off)
    off += 2
    if len(data) < off + 12 * nch:
        raise FormatError("truncated chunk table")
    ents = [struct.unpack_from("<III", data, off + 12 * i) for i in range(nch)]
    off += 12 * nch
    chunks = []
    for n, bits, ln in ents:
        if ln != (bits + 7) // 8:
            raise FormatError("stream_len != ceil(bit_count/8)")
        if off + ln > len(data):
            raise FormatError("truncated stream")
        chunks.append((n, bits, bytes(data[off:off + ln])))
        off += ln
    if off != len(data):
        raise FormatError("trailing bytes")
    return flags, tau_milli, regs, method, payload, chunks


def compress_file(data: bytes, weights, prm):
    """NC06 of arbitrary bytes with the oracle text pipeline."""
    from .compressor import compress
    from .container import read_nc05
    regs = segment(data)
    if len(regs) > 0xFFFF:
        regs = [(BINARY, len(data))]
    text, binary = split(data, regs)
    method, payload = blob_encode(binary)
    _, _, chunks = read_nc05(compress(text, weights, prm))
    return write_nc06(prm.flags, prm.tau_milli, regs, method, payload, chunks)


def decompress_file(blob: bytes, weights, prm):
    from .compressor import decompress
    from .container import write_nc05
    flags, tau_milli, regs, method, payload, chunks = read_nc06(blob)
    text = decompress(write_nc05(flags, tau_milli, chunks), weights, prm)
    binary = blob_decode(method, payload)
    out, ti, bi = [], 0, 0
    for k, ln in regs:
        if k == TEXT:
            out.append(text[ti:ti + ln])
            ti += ln
        else:
            out.append(binary[bi:bi + ln])
            bi += ln
    if ti != len(text) or bi != len(binary):
        raise FormatError("entry lengths do not match the sections")
    return b"".join(out)
