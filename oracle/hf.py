"""HF-format checkpoints for the oracle.
CPU ORACLE -- test infrastructure only (see oracle/__init__.py).

Own readers, independent of libnc's: config.json (json), model.safetensors (the 8-byte
header length, the JSON header, raw F32 / F16 / BF16 data -> fp64 with numpy), and the
tokenizer through the HF ``tokenizers`` library itself (a library routine: the paper
tokenizes with SmolLM2's HF tokenizer).  ``HfWeights`` has the attributes of
oracle.ncw.Weights, so oracle.lm.LM and the pipeline run on it unchanged; the vocabulary
bytes come from the GPT-2 byte-level alphabet (bytes_to_unicode, written out below).

Reading D35: special tokens are never produced from input text; the tokenizer's input is
UTF-8 text (invalid UTF-8 is outside what the HF library accepts, so the oracle rejects it).
"""
import json
import struct
from pathlib import Path

import numpy as np


def bytes_to_unicode():
    """GPT-2's byte-level alphabet: printable Latin-1 bytes map to themselves, the other 68
    bytes to U+0100.. in byte order."""
    bs = list(range(ord("!"), ord("~") + 1)) + list(range(0xA1, 0xAC + 1)) + list(range(0xAE, 0xFF + 1))
    cs = bs[:]
    n = 0
    for b in range(256):
        if b not in bs:
            bs.append(b)
            cs.append(256 + n)
            n += 1
    return {b: chr(c) for b, c in zip(bs, cs)}


def read_safetensors(path):
    raw = Path(path).read_bytes()
    (hn,) = struct.unpack_from("<Q", raw, 0)
    hdr = json.loads(raw[8:8 + hn])
    base = 8 + hn
    out = {}
    for name, t in hdr.items():
        if name == "__metadata__":
            continue
        b0, b1 = t["data_offsets"]
        buf = raw[base + b0:base + b1]
        if t["dtype"] == "F32":
            a = np.frombuffer(buf, "<f4").astype(np.float64)
        elif t["dtype"] == "BF16":
            a = (np.frombuffer(buf, "<u2").astype(np.uint32) << 16).view("<f4").astype(np.float64)
        elif t["dtype"] == "F16":
            a = np.frombuffer(buf, "<f2").astype(np.float64)
        else:
            raise ValueError(t["dtype"])
        out[name] = a.reshape(t["shape"])
    return out


class HfTokenizer:
    """encode(bytes) -> ids with the HF tokenizers library; decode(ids) -> bytes."""

    def __init__(self, path, vocab_bytes):
        from tokenizers import Tokenizer
        self.tok = Tokenizer.from_file(str(path))
        self.vocab = vocab_bytes

    def encode(self, data: bytes):
        return self.tok.encode(data.decode("utf-8"), add_special_tokens=False).ids

    def decode(self, ids) -> bytes:
        return b"".join(self.vocab[i] for i in ids)


class HfWeights:
    def __init__(self, model_dir):
        d = Path(model_dir)
        cfg = json.loads((d / "config.json").read_text())
        self.d, self.n_layers = cfg["hidden_size"], cfg["num_hidden_layers"]
        self.H = cfg["num_attention_heads"]
        self.KV = cfg.get("num_key_value_heads", self.H)
        self.dh = cfg.get("head_dim", self.d // self.H)
        self.d_ff, self.V = cfg["intermediate_size"], cfg["vocab_size"]
        self.eps, self.rope_theta = cfg["rms_norm_eps"], cfg.get("rope_theta", 10000.0)
        self.bos = cfg.get("bos_token_id", 0)
        assert cfg.get("tie_word_embeddings")
        t = read_safetensors(d / "model.safetensors")
        self.embed = t["model.embed_tokens.weight"]
        self.layers = []
        for i in range(self.n_layers):
            p = f"model.layers.{i}."
            self.layers.append(dict(
                attn_norm=t[p + "input_layernorm.weight"], wq=t[p + "self_attn.q_proj.weight"],
                wk=t[p + "self_attn.k_proj.weight"], wv=t[p + "self_attn.v_proj.weight"],
                wo=t[p + "self_attn.o_proj.weight"], mlp_norm=t[p + "post_attention_layernorm.weight"],
                wg=t[p + "mlp.gate_proj.weight"], wu=t[p + "mlp.up_proj.weight"], wd=t[p + "mlp.down_proj.weight"]))
        self.final_norm = t["model.norm.weight"]
        tj = json.loads((d / "tokenizer.json").read_text())
        inv = {c: b for b, c in bytes_to_unicode().items()}
        vocab = [b""] * self.V
        for s, i in tj["model"]["vocab"].items():
            vocab[i] = bytes(inv[c] for c in s)
        specials = [a for a in tj.get("added_tokens", [])]
        for a in specials:
            vocab[a["id"]] = a["content"].encode()
        self.n_special = sum(1 for a in specials if a.get("special"))
        self.vocab = vocab
        self.tokenizer = HfTokenizer(d / "tokenizer.json", vocab)
