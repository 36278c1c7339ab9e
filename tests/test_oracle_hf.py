"""NEXT-2 pins: HF-format checkpoints and the
byte-level BPE tokenizer.

* The oracle's own safetensors / config reader (oracle/hf.py) reproduces HF transformers'
  LlamaForCausalLM.from_pretrained on the same directory (a library routine), logits 1e-5.
* The oracle tokenizer IS the HF tokenizers library; its vocabulary-bytes table (GPT-2
  byte-level alphabet written out) is pinned by exact round trips.
* libnc's C++ BPE (nc_host_bpe_encode: hand-written GPT-2 pre-tokenizer + ranked merges)
  gives the same ids as the HF library on synthetic prose, MediaWiki text with non-ASCII
  UTF-8, and edge strings (contractions, whitespace runs, digits, punctuation, scripts);
  and exact round trips on arbitrary bytes (invalid UTF-8 included, reading D35)."""
import numpy as np
import pytest
import torch

import paper_2602_19626_b200 as nc
from oracle.hf import HfWeights, bytes_to_unicode
from oracle.lm import LM, window_start


@pytest.fixture(scope="module")
def hf_tiny():
    from synth.hf import ensure_hf_model
    return ensure_hf_model("hf-tiny")


def test_bytes_to_unicode_alphabet():
    m = bytes_to_unicode()
    assert len(m) == 256 and len(set(m.values())) == 256
    assert m[ord("A")] == "A" and m[ord(" ")] == "Ġ" and m[ord("\n")] == "Ċ" and m[0] == "Ā"


def test_oracle_hf_weights_match_transformers(hf_tiny):
    from transformers import LlamaForCausalLM
    w = HfWeights(hf_tiny)
    assert np.abs(w.final_norm - 1).max() > 0.1                       # non-unit gains are exercised
    m = LlamaForCausalLM.from_pretrained(str(hf_tiny), torch_dtype=torch.float64).eval()
    L, C, n = 16, 4, 40
    x = list(np.random.default_rng(3).integers(0, w.V, n))
    ours = LM(w).forward_blocked(x, L, C)
    mask = torch.full((1, 1, n, n), float("-inf"), dtype=torch.float64)
    for j in range(n):
        mask[0, 0, j, window_start(j, L, C):j + 1] = 0.0
    with torch.no_grad():
        hf = m(torch.tensor([x]), attention_mask=mask).logits[0].numpy()
    assert np.abs(hf - ours).max() / np.abs(ours).max() < 1e-5


def test_oracle_hf_tokenizer_roundtrip(hf_tiny):
    from synth import make_text
    w = HfWeights(hf_tiny)
    for data in (make_text("alice", 5000, 1), make_text("enwik", 5000, 2), "naïve — 'twas 42 €\n\n\t x".encode()):
        ids = w.tokenizer.encode(data)
        assert w.tokenizer.decode(ids) == data and all(i >= w.n_special for i in ids)


EDGE = ["", "a", " ", "  ", "\n\n\nword", "hello  world", "it's they're we've I'm you'll he'd 'S",
        "x123y 4567 8", "tab\tsep\n  two spaces\n", "¡Hola! ¿qué tal? — “quoted” ‘single’",
        "αβγ δεζ 中文字符 日本語 한국어", "emoji 😀👍🏽 done", "mixed123abc   \n\t  end  ",
        "a'b 'c ' '' '''", "…!!!??.,;:", " nbsp emsp", "trailing spaces   "]


@pytest.mark.parametrize("text", EDGE)
def test_cpp_bpe_equals_hf_tokenizers_edges(hf_tiny, text):
    from tokenizers import Tokenizer
    tok = Tokenizer.from_file(str(hf_tiny / "tokenizer.json"))
    ref = tok.encode(text, add_special_tokens=False).ids
    assert nc.nc_host_bpe_encode(hf_tiny / "tokenizer.json", 512, text.encode()) == ref


@pytest.mark.parametrize("kind,seed", [("alice", 5), ("enwik", 6), ("enwik", 7)])
def test_cpp_bpe_equals_hf_tokenizers_text(hf_tiny, kind, seed):
    from tokenizers import Tokenizer
    from synth import make_text
    tok = Tokenizer.from_file(str(hf_tiny / "tokenizer.json"))
    data = make_text(kind, 60000, seed)
    ref = tok.encode(data.decode(), add_special_tokens=False).ids
    assert nc.nc_host_bpe_encode(hf_tiny / "tokenizer.json", 512, data) == ref


def test_cpp_bpe_roundtrip_arbitrary_bytes(hf_tiny):
    w = HfWeights(hf_tiny)
    rng = np.random.default_rng(9)
    for _ in range(20):
        data = bytes(rng.integers(0, 256, int(rng.integers(0, 3000))).astype(np.uint8))
        ids = nc.nc_host_bpe_encode(hf_tiny / "tokenizer.json", 512, data)
        assert b"".join(w.vocab[i] for i in ids) == data
