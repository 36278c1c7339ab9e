"""Oracle pins for the LM forward and window semantics.

(i)  HF transformers LlamaForCausalLM (fp64, same tensors, 4-D additive window
     mask) reproduces the oracle's blocked forward for every row -- a textbook
     library routine independent of our code.
(ii) literal llama.cpp-style rm/shift incremental loop == blocked masked pass.
(iii) 1-layer model: row j is invariant to tokens before w(j).
(iv) window arithmetic of S:355 and P:486-500.
"""
import numpy as np
import pytest
import torch

from oracle.lm import LM, window_start


def test_window_arithmetic():
    L, C = 2048, 512
    assert [window_start(j, L, C) for j in (0, 2046, 2047)] == [0, 0, 0]
    # after 2048 advances one more -> context [512..2048]
    assert window_start(2048, L, C) == 512
    ctx = [j - window_start(j, L, C) + 1 for j in range(L, 6 * L)]
    assert min(ctx) == L - C + 1 and max(ctx) == L
    # slides happen every C rows once past L (D10: "C advances", not L-C)
    slides = [j for j in range(1, 6 * L) if window_start(j, L, C) != window_start(j - 1, L, C)]
    assert slides[0] == L and all(b - a == C for a, b in zip(slides, slides[1:]))
    assert window_start(8, 8, 2) == 2 and window_start(9, 8, 2) == 2 and window_start(10, 8, 2) == 4


@pytest.mark.parametrize("L,C,n", [(8, 2, 30), (16, 4, 45)])
def test_literal_equals_blocked(tiny_weights, L, C, n):
    lm = LM(tiny_weights)
    x = list(np.random.default_rng(n).integers(0, tiny_weights.V, n))
    a = lm.forward_blocked(x, L, C, rows_per_block=7)
    b = lm.forward_literal(x, L, C)
    assert np.abs(a - b).max() < 1e-12 * max(1.0, np.abs(a).max())


def _hf_model(w):
    from transformers import LlamaConfig, LlamaForCausalLM
    cfg = LlamaConfig(vocab_size=w.V, hidden_size=w.d, intermediate_size=w.d_ff,
                      num_hidden_layers=w.n_layers, num_attention_heads=w.H,
                      num_key_value_heads=w.KV, head_dim=w.dh, rms_norm_eps=w.eps,
                      rope_parameters={"rope_theta": w.rope_theta, "rope_type": "default"},
                      tie_word_embeddings=True, attention_bias=False, mlp_bias=False,
                      max_position_embeddings=4096)
    cfg._attn_implementation = "eager"
    m = LlamaForCausalLM(cfg).double().eval()
    sd = {"model.embed_tokens.weight": w.embed, "model.norm.weight": w.final_norm}
    for i, lw in enumerate(w.layers):
        p = f"model.layers.{i}."
        sd.update({p + "input_layernorm.weight": lw["attn_norm"],
                   p + "self_attn.q_proj.weight": lw["wq"], p + "self_attn.k_proj.weight": lw["wk"],
                   p + "self_attn.v_proj.weight": lw["wv"], p + "self_attn.o_proj.weight": lw["wo"],
                   p + "post_attention_layernorm.weight": lw["mlp_norm"],
                   p + "mlp.gate_proj.weight": lw["wg"], p + "mlp.up_proj.weight": lw["wu"],
                   p + "mlp.down_proj.weight": lw["wd"]})
    with torch.no_grad():
        for k, v in m.state_dict().items():
            if k in sd:
                v.copy_(torch.from_numpy(np.ascontiguousarray(sd[k])))
            elif k == "lm_head.weight":
                v.copy_(torch.from_numpy(w.embed))
    return m


@pytest.mark.parametrize("wname", ["tiny_weights", "tinyg_weights"])
def test_hf_llama_window_mask_matches_blocked(request, wname):
    """unit gains (D16) and non-unit gains U(0.5, 1.5) (tiny-g): a wrong gain axis or a
    dropped gain in the oracle fails the second case."""
    w = request.getfixturevalue(wname)
    if wname == "tinyg_weights":
        assert np.abs(w.final_norm - 1).max() > 0.1 and np.abs(w.layers[0]["attn_norm"] - 1).max() > 0.1
    L, C, n = 16, 4, 40
    x = list(np.random.default_rng(3).integers(0, w.V, n))
    ours = LM(w).forward_blocked(x, L, C)
    m = _hf_model(w)
    mask = torch.full((1, 1, n, n), float("-inf"), dtype=torch.float64)
    for j in range(n):
        mask[0, 0, j, window_start(j, L, C):j + 1] = 0.0
    with torch.no_grad():
        hf = m(torch.tensor([x]), attention_mask=mask).logits[0].numpy()
    # HF's RMSNorm computes in fp32 even in a float64 model -> ~1e-7 relative noise
    err = np.abs(hf - ours).max() / np.abs(ours).max()
    assert err < 1e-5, err
    # and the window matters: the plain causal model differs on rows >= L
    with torch.no_grad():
        causal = m(torch.tensor([x])).logits[0].numpy()
    assert np.abs(causal[:L] - ours[:L]).max() / np.abs(ours).max() < 1e-5
    assert np.abs(causal[L:] - ours[L:]).max() / np.abs(ours).max() > 1e-3


def test_one_layer_row_invariant_to_dropped_tokens(tiny1_weights):
    w = tiny1_weights
    L, C, n = 8, 2, 24
    rng = np.random.default_rng(4)
    x = list(rng.integers(0, w.V, n))
    a = LM(w).forward_blocked(x, L, C)
    j = 20
    y = list(x)
    for k in range(window_start(j, L, C)):
        y[k] = int(rng.integers(w.V))
    b = LM(w).forward_blocked(y, L, C)
    assert np.abs(a[j] - b[j]).max() < 1e-12


def test_two_layer_retained_kv_is_not_refresh(tiny_weights):
    """D9: with >= 2 layers the retained-KV semantics differ from re-evaluating the window."""
    w = tiny_weights
    L, C, n = 8, 2, 16
    x = list(np.random.default_rng(5).integers(0, w.V, n))
    a = LM(w).forward_blocked(x, L, C)
    j = 12
    s = window_start(j, L, C)
    fresh = LM(w).forward_blocked(x[s:j + 1], 10 ** 6, 1)[-1]
    assert np.abs(a[j] - fresh).max() > 1e-6


def test_rope_relative_invariance():
    from oracle.lm import apply_rope, rope_tables
    rng = np.random.default_rng(6)
    q = rng.standard_normal((1, 1, 64))
    k = rng.standard_normal((1, 1, 64))
    def score(pq, pk):
        cq, sq = rope_tables([pq], 64, 1e5)
        ck, sk = rope_tables([pk], 64, 1e5)
        return float((apply_rope(q, cq, sq) * apply_rope(k, ck, sk)).sum())
    assert abs(score(10, 3) - score(510, 503)) < 1e-10
    assert abs(score(10, 3) - score(10, 4)) > 1e-6


# ---------------------------------------------------------------- NEXT-4 variants ---
@pytest.mark.parametrize("lmax", [16, 15])
def test_refresh_literal_equals_blocked(tiny_weights, lmax):
    """refresh semantics (the naive re-evaluation of P:489-492): the literal loop that clears
    the cache and re-evaluates the survivors on every slide == one fresh causal pass per
    window block (1e-12); for L_max = L and L - 1 (D10)."""
    lm = LM(tiny_weights)
    x = list(np.random.default_rng(40 + lmax).integers(0, tiny_weights.V, 45))
    a = lm.forward_literal(x, 16, 4, lmax=lmax, refresh=True)
    b = lm.forward_refresh_blocked(x, 16, 4, lmax=lmax)
    assert np.abs(a - b).max() < 1e-12 * max(1.0, np.abs(a).max())


@pytest.mark.parametrize("lmax", [16, 15])
def test_refresh_equals_hf_fresh_window(tiny_weights, lmax):
    """S:361's window equivalence, which holds exactly under refresh semantics: row j equals
    a FRESH evaluation of the surviving window x[w(j) .. j] -- computed here by HF
    LlamaForCausalLM (a library routine, fp64) on that slice alone."""
    w = tiny_weights
    x = list(np.random.default_rng(7).integers(0, w.V, 40))
    ours = LM(w).forward_refresh_blocked(x, 16, 4, lmax=lmax)
    m = _hf_model(w)
    for j in (0, 5, lmax - 1, lmax, lmax + 1, 22, 30, 39):
        s = window_start(j, lmax, 4)
        with torch.no_grad():
            hf = m(torch.tensor([x[s:j + 1]])).logits[0, -1].numpy()
        assert np.abs(hf - ours[j]).max() / np.abs(ours[j]).max() < 1e-5, j
    # and it differs from retained-KV semantics once a slide has happened (>= 2 layers, D9)
    ret = LM(w).forward_blocked(x, lmax, 4)
    assert np.abs(ret[:lmax] - ours[:lmax]).max() < 1e-12
    assert np.abs(ret[lmax + 4:] - ours[lmax + 4:]).max() > 1e-6


def test_lmax_minus_one_window_arithmetic():
    """L_max = L - 1 (D10's other reading): the first slide happens one row earlier, context
    <= L - 1, slides every C rows after it."""
    L, C = 2048, 512
    lmax = L - 1
    assert window_start(L - 2, lmax, C) == 0 and window_start(L - 1, lmax, C) == C
    ctx = [j - window_start(j, lmax, C) + 1 for j in range(lmax, 6 * L)]
    assert min(ctx) == lmax - C + 1 and max(ctx) == lmax
    slides = [j for j in range(1, 6 * L) if window_start(j, lmax, C) != window_start(j - 1, lmax, C)]
    assert slides[0] == L - 1 and all(b - a == C for a, b in zip(slides, slides[1:]))


def test_lmax_minus_one_literal_equals_blocked_and_hf(tiny_weights):
    """retained KV with L_max = L - 1: the literal rm/shift loop (slide when the cache would
    exceed L - 1) == the blocked pass with w(j) on L_max == HF with the 4-D window mask."""
    w = tiny_weights
    L, C, n = 16, 4, 40
    x = list(np.random.default_rng(9).integers(0, w.V, n))
    a = LM(w).forward_literal(x, L, C, lmax=L - 1)
    b = LM(w).forward_blocked(x, L - 1, C)
    assert np.abs(a - b).max() < 1e-12 * max(1.0, np.abs(a).max())
    mask = torch.full((1, 1, n, n), float("-inf"), dtype=torch.float64)
    for j in range(n):
        mask[0, 0, j, window_start(j, L - 1, C):j + 1] = 0.0
    with torch.no_grad():
        hf = _hf_model(w)(torch.tensor([x]), attention_mask=mask).logits[0].numpy()
    assert np.abs(hf - b).max() / np.abs(b).max() < 1e-5
