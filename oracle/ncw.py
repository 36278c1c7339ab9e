"""NCW1 weight-file reader for the oracle (own parser; format documented in
synth/weights.py).  Returns fp64 arrays (the paper runs the model in
FP32; the oracle runs it in fp64 so that it is the exact reference)."""
import struct

import numpy as np


class Weights:
    def __init__(self, path):
        raw = open(path, "rb").read()
        if raw[:4] != b"NCW1":
            raise ValueError("not an NCW1 file")
        (ver, self.n_layers, self.d, self.H, self.KV, self.dh, self.d_ff, self.V, self.bos,
         self.n_special) = struct.unpack_from("<10I", raw, 4)
        self.rope_theta, self.eps = struct.unpack_from("<dd", raw, 44)
        assert ver == 1
        off = 64

        def take(*shape):
            nonlocal off
            n = int(np.prod(shape))
            a = np.frombuffer(raw, dtype="<f4", count=n, offset=off).reshape(shape)
            off += 4 * n
            return a.astype(np.float64)

        d, H, KV, dh, f, V = self.d, self.H, self.KV, self.dh, self.d_ff, self.V
        self.embed = take(V, d)
        self.layers = []
        for _ in range(self.n_layers):
            self.layers.append(dict(
                attn_norm=take(d), wq=take(H * dh, d), wk=take(KV * dh, d), wv=take(KV * dh, d),
                wo=take(d, H * dh), mlp_norm=take(d), wg=take(f, d), wu=take(f, d), wd=take(d, f)))
        self.final_norm = take(d)
        (nv,) = struct.unpack_from("<I", raw, off)
        off += 4
        assert nv == V
        vocab = []
        for _ in range(nv):
            (ln,) = struct.unpack_from("<H", raw, off)
            off += 2
            vocab.append(bytes(raw[off:off + ln]))
            off += ln
        self.vocab = vocab
        assert off == len(raw)
