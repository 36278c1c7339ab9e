"""HF-format model directories for the NEXT-2 tests.

The real SmolLM2-135M checkpoint and tokenizer are not on disk (no network), so this writes
a stand-in with the SAME file formats:

* ``tokenizer.json``: a byte-level BPE trained with the HF ``tokenizers`` library on seeded
  synthetic text (alice- and enwik-shaped, with non-ASCII UTF-8), with SmolLM2's pipeline:
  pre-tokenizer Sequence[Digits(individual_digits=True), ByteLevel(add_prefix_space=False)],
  ByteLevel decoder, special tokens <|endoftext|> (id 0, BOS), <|im_start|>, <|im_end|>;
* ``config.json``: LlamaConfig fields of the shape (tie_word_embeddings = true, theta 1e5);
* ``model.safetensors``: random-init weights (N(0, 1/24^2), norm gains U(0.5, 1.5)) stored
  as BF16 like the released checkpoint, HF Llama tensor names.

No arithmetic of the compression method lives here (cf. synth/__init__.py).
"""
import json
from pathlib import Path

import numpy as np

from .configs import SHAPES
from .text import make_text
from .weights import cache_dir

HF_SHAPES = {
    # (base shape, BPE vocabulary size the trainer aims for)
    "hf-smollm2-2l": ("smollm2-2l", 49152),
    "hf-tiny": ("tiny", 512),
}


def _train_tokenizer(vocab_size: int, seed: int = 2602):
    from tokenizers import Tokenizer, decoders, models, pre_tokenizers, trainers
    tok = Tokenizer(models.BPE())
    tok.pre_tokenizer = pre_tokenizers.Sequence([pre_tokenizers.Digits(individual_digits=True),
                                                 pre_tokenizers.ByteLevel(add_prefix_space=False, use_regex=True)])
    tok.decoder = decoders.ByteLevel()
    trainer = trainers.BpeTrainer(vocab_size=vocab_size, min_frequency=2,
                                  special_tokens=["<|endoftext|>", "<|im_start|>", "<|im_end|>"],
                                  initial_alphabet=pre_tokenizers.ByteLevel.alphabet(), show_progress=False)
    corpus = [make_text("alice", 1_500_000, seed).decode(), make_text("enwik", 1_500_000, seed + 1).decode()]
    lines = [ln for doc in corpus for ln in doc.split("\n")]
    tok.train_from_iterator(lines, trainer)
    return tok


def write_hf_model(out_dir: Path, name: str):
    import torch
    from safetensors.torch import save_file
    base, bpe_vocab = HF_SHAPES[name]
    s = SHAPES[base]
    out_dir.mkdir(parents=True, exist_ok=True)
    tok = _train_tokenizer(bpe_vocab)
    assert tok.get_vocab_size() <= s.vocab
    tok.save(str(out_dir / "tokenizer.json"))
    cfg = {"architectures": ["LlamaForCausalLM"], "model_type": "llama", "hidden_size": s.d_model,
           "num_hidden_layers": s.n_layers, "num_attention_heads": s.n_heads, "num_key_value_heads": s.n_kv_heads,
           "head_dim": s.head_dim, "intermediate_size": s.d_ff, "vocab_size": s.vocab, "rms_norm_eps": s.rms_eps,
           "rope_theta": s.rope_theta, "tie_word_embeddings": True, "hidden_act": "silu", "bos_token_id": 0,
           "eos_token_id": 0, "max_position_embeddings": 8192, "attention_bias": False, "mlp_bias": False,
           "torch_dtype": "bfloat16"}
    (out_dir / "config.json").write_text(json.dumps(cfg, indent=1))
    rng = np.random.default_rng(s.weight_seed + 100)
    d, H, KV, dh, f, V = s.d_model, s.n_heads, s.n_kv_heads, s.head_dim, s.d_ff, s.vocab

    def mat(*shape):
        return torch.from_numpy((rng.standard_normal(shape) * s.init_std).astype(np.float32)).to(torch.bfloat16)

    def gain(n):
        return torch.from_numpy(rng.uniform(0.5, 1.5, n).astype(np.float32)).to(torch.bfloat16)

    t = {"model.embed_tokens.weight": mat(V, d)}
    for i in range(s.n_layers):
        p = f"model.layers.{i}."
        t[p + "input_layernorm.weight"] = gain(d)
        t[p + "self_attn.q_proj.weight"] = mat(H * dh, d)
        t[p + "self_attn.k_proj.weight"] = mat(KV * dh, d)
        t[p + "self_attn.v_proj.weight"] = mat(KV * dh, d)
        t[p + "self_attn.o_proj.weight"] = mat(d, H * dh)
        t[p + "post_attention_layernorm.weight"] = gain(d)
        t[p + "mlp.gate_proj.weight"] = mat(f, d)
        t[p + "mlp.up_proj.weight"] = mat(f, d)
        t[p + "mlp.down_proj.weight"] = mat(d, f)
    t["model.norm.weight"] = gain(d)
    save_file(t, str(out_dir / "model.safetensors"), metadata={"format": "pt"})


def ensure_hf_model(name: str) -> Path:
    d = cache_dir() / f"{name}.hf"
    if not (d / "model.safetensors").exists():
        tmp = cache_dir() / f"{name}.hf.tmp"
        write_hf_model(tmp, name)
        if d.exists():
            import shutil
            shutil.rmtree(d)
        tmp.rename(d)
    return d
