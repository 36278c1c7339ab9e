"""NC05 container.

Header (9 bytes): b"NC05", flags u8 (bit0 N-gram, bit1 adaptive head, bit2
skip; bits 3-7 zero), temperature u16 LE = round(tau*1000), chunk_count u16 LE;
then chunk_count x {token_count u32, bit_count u32, stream_len u32 =
ceil(bit_count/8)}; then the streams concatenated in chunk order.
"""
import struct


class FormatError(ValueError):
    pass


def write_nc05(flags, tau_milli, chunks):
    """chunks: list of (token_count, bit_count, stream_bytes)."""
    if len(chunks) > 0xFFFF:
        raise FormatError("chunk overflow")
    out = [b"NC05", struct.pack("<BHH", flags, tau_milli, len(chunks))]
    for n, bits, s in chunks:
        if len(s) != (bits + 7) // 8:
            raise FormatError("stream_len != ceil(bit_count/8)")
        out.append(struct.pack("<III", n, bits, len(s)))
    out += [s for _, _, s in chunks]
    return b"".join(out)


def read_nc05(data: bytes):
    if len(data) < 9:
        raise FormatError("truncated header")
    if data[:4] != b"NC05":
        raise FormatError("bad magic")
    flags, tau_milli, n = struct.unpack_from("<BHH", data, 4)
    if flags & ~0x07:
        raise FormatError("reserved flag bits set")
    off = 9
    if len(data) < off + 12 * n:
        raise FormatError("truncated chunk table")
    ents = [struct.unpack_from("<III", data, off + 12 * i) for i in range(n)]
    off += 12 * n
    chunks = []
    for tok, bits, ln in ents:
        if ln != (bits + 7) // 8:
            raise FormatError("stream_len != ceil(bit_count/8)")
        if off + ln > len(data):
            raise FormatError("truncated stream")
        chunks.append((tok, bits, bytes(data[off:off + ln])))
        off += ln
    if off != len(data):
        raise FormatError("trailing bytes")
    return flags, tau_milli, chunks
