"""Parallel chunking ("splits the input text into N roughly equal
chunks (at newline boundaries)").

Reading: for i = 1..N-1 the cut is just after the first b'\\n' at or after
max(i*ceil(len/N), previous cut); if there is none the cut is a hard split at
that target.  Cuts at or past the end are dropped, so there are at most N
chunks and their concatenation is the input.  Empty input gives one empty chunk
("chunk_count = N' <= 1").
"""


def split_chunks(data: bytes, n_chunks: int):
    n = len(data)
    if n_chunks <= 1 or n == 0:
        return [bytes(data)]
    step = -(-n // n_chunks)
    cuts = [0]
    for i in range(1, n_chunks):
        target = max(i * step, cuts[-1])
        if target >= n:
            break
        j = data.find(b"\n", target)
        cut = j + 1 if j >= 0 else target
        if cut >= n:
            break
        if cut > cuts[-1]:
            cuts.append(cut)
    ends = cuts[1:] + [n]
    return [bytes(data[a:b]) for a, b in zip(cuts, ends)]
