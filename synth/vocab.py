"""Synthetic token vocabulary.

ids 0..2 are specials (0 = BOS "<|endoftext|>", as SmolLM2's id 0; D13), ids 3..258
are the 256 single bytes (so every byte string tokenizes), and the rest are
lexicon / markup / number / syllable strings up to the requested size V.
The real SmolLM2 BPE is unavailable offline (NEXT-2).  The tokenizer itself
(greedy longest match) is implemented separately by the oracle and by the C++
runtime; this module only lists the strings.
"""
from .text import lexicon, syllables, NON_ASCII

SPECIALS = [b"<|endoftext|>", b"<|im_start|>", b"<|im_end|>"]
N_SPECIAL = 3
BYTE_BASE = 3

_PUNCT = [",", ".", ";", ":", "!", "?", '"', "'", "(", ")", "-", "--", "|", "*", "="]
_MARKUP = ["[[", "]]", "{{", "}}", "'''", "''", "==", " ==", "== ", "===", "&lt;", "&gt;",
           "&amp;", "&quot;", "&lt;ref&gt;", "&lt;/ref&gt;", "<page>", "</page>", "<title>",
           "</title>", "<id>", "</id>", "<revision>", "</revision>", "<timestamp>",
           "</timestamp>", '<text xml:space="preserve">', "</text>", "[[Category:", "\n* [[",
           "* [[", "]]\n", "}}\n", " ==\n", "\n== ", "  <page>\n", "    <title>", "    <id>",
           "    <revision>\n", "      <id>", "      <timestamp>", "      <text",
           "</text>\n", "    </revision>\n", "  </page>\n", "</title>\n", "</id>\n",
           "</timestamp>\n", "CHAPTER ", "http://", "www.", ".com", ".org", "<mediawiki"]


def make_vocab(V: int):
    """Return the list of V byte strings; index = token id."""
    if V < 259 + 16:
        raise ValueError("vocab too small")
    out = list(SPECIALS) + [bytes([b]) for b in range(256)]
    seen = set(out)

    def add(s):
        b = s.encode("utf-8") if isinstance(s, str) else s
        if len(out) < V and b not in seen and 1 < len(b) <= 48:
            seen.add(b)
            out.append(b)

    words = lexicon()
    syl = syllables()
    # punctuation / whitespace combos first (highest frequency in prose)
    for p in _PUNCT:
        for a, z in (("", " "), (" ", ""), ("", "\n"), ("", "\n\n"), (" ", " ")):
            add(a + p + z)
    for a in ('."', ',"', '?"', '!"', ' "', '" ', '."\n', '.\n\n', '\n\n', '\n', '  ', '    '):
        add(a)
    for m in _MARKUP:
        add(m)
    for c in NON_ASCII:
        add(c)
    # words in frequency order, four casings/spacings each
    for w in words:
        add(" " + w)
        add(w)
        add(" " + w.capitalize())
        add(w.capitalize())
        if len(out) >= V:
            break
    for n in range(1000):
        add(str(n))
        add(" " + str(n))
    for y in range(1800, 2026):
        add(str(y))
        add(" " + str(y))
    for w in words:
        add(w + ",")
        add(w + ".")
        add("[[" + w)
        add(w.upper())
    for s in syl:
        add(s)
        add(" " + s)
        add(s.capitalize())
    i = 0
    while len(out) < V:
        a, b = syl[i % len(syl)], syl[(i * 7919 + 13) % len(syl)]
        add(a + b)
        add(" " + a + b)
        i += 1
        if i > 10_000_000:
            raise RuntimeError("vocab fill did not converge")
    assert len(out) == V
    return out
