"""alice29- and enwik8-shaped synthetic text (SURVEY.md §8(d) "Synthetic inputs").

alice-shaped: ASCII prose (bytes 10, 32-126); an order-2 word Markov chain over a
Zipf(1.07) lexicon of ~8K seeded-syllable words; sentences of 5-25 words with
dialogue quotes and punctuation; lines wrapped at <=72 characters; blank lines
between paragraphs; a chapter heading every ~15 KB.

enwik-shaped: MediaWiki XML pages wrapping the same prose, with [[links]],
{{templates}}, '''bold''', == headings ==, * lists, &lt;ref&gt; entities, numbers,
dates and ~1-2 % non-ASCII UTF-8 characters.

mixed: an arbitrary-file-shaped byte stream (text segments alternating with binary
segments) for the NC06 hybrid format.

Everything is a pure function of (kind, n_bytes, seed).
"""
import numpy as np

_ONSETS = ["", "b", "c", "d", "f", "g", "h", "j", "k", "l", "m", "n", "p", "r", "s", "t",
           "v", "w", "y", "z", "ch", "sh", "th", "wh", "br", "cr", "dr", "fr", "gr", "pr",
           "tr", "bl", "cl", "fl", "gl", "pl", "sl", "sp", "st", "sw", "qu"]
_NUCLEI = ["a", "e", "i", "o", "u", "ea", "ee", "oo", "ou", "ai", "ie", "oa", "y"]
_CODAS = ["", "", "", "", "", "", "", "n", "r", "s", "t", "l", "d", "m", "ng", "ck", "st", "nd", "rt", "ll"]

ZIPF_S = 1.07
N_WORDS = 8000
NON_ASCII = ["é", "ü", "ö", "ñ", "ç", "—", "–", "’", "“", "”", "€", "°", "ß", "å", "ø"]


def syllables(seed: int = 11, n: int = 400):
    rng = np.random.default_rng(seed)
    out, seen = [], set()
    while len(out) < n:
        s = (_ONSETS[rng.integers(len(_ONSETS))] + _NUCLEI[rng.integers(len(_NUCLEI))]
             + _CODAS[rng.integers(len(_CODAS))])
        if s not in seen:
            seen.add(s)
            out.append(s)
    return out


def lexicon(seed: int = 12, n: int = N_WORDS):
    """~8K distinct lowercase words built from seeded syllables; index = Zipf rank."""
    rng = np.random.default_rng(seed)
    syl = syllables()
    words, seen = [], set()
    # a few very short function-like words first (highest frequency ranks)
    for w in ["the", "and", "to", "a", "of", "it", "she", "said", "in", "was", "you", "i",
              "as", "that", "her", "at", "on", "all", "with", "had", "but", "for", "so", "be"]:
        words.append(w)
        seen.add(w)
    while len(words) < n:
        k = 1 + min(2, int(rng.geometric(0.7)) - 1)
        w = "".join(syl[int(rng.integers(len(syl)))] for _ in range(k))
        if 1 < len(w) <= 14 and w not in seen:
            seen.add(w)
            words.append(w)
    return words


def _zipf_cdf(n: int, s: float = ZIPF_S):
    w = 1.0 / np.arange(1, n + 1, dtype=np.float64) ** s
    c = np.cumsum(w)
    return c / c[-1]


class _Prose:
    """Order-2 word Markov chain: P(w | w2, w1) mixes successor lists of w1 and w2
    with the Zipf unigram."""

    def __init__(self, seed: int):
        self.rng = np.random.default_rng(seed)
        self.words = lexicon()
        n = len(self.words)
        self.cdf = _zipf_cdf(n)
        srng = np.random.default_rng(seed ^ 0x5EED)
        # 12 successors per word drawn from the Zipf unigram
        self.succ = np.searchsorted(self.cdf, srng.random((n, 12)))
        self.succ_cdf = _zipf_cdf(12, 1.3)
        self.buf = self.rng.random(1 << 16)
        self.pos = 0

    def u(self) -> float:
        if self.pos >= len(self.buf):
            self.buf = self.rng.random(1 << 16)
            self.pos = 0
        v = self.buf[self.pos]
        self.pos += 1
        return v

    def unigram(self) -> int:
        return int(np.searchsorted(self.cdf, self.u()))

    def next_word(self, w2: int, w1: int) -> int:
        r = self.u()
        if w1 >= 0 and r < 0.55:
            return int(self.succ[w1, np.searchsorted(self.succ_cdf, self.u())])
        if w2 >= 0 and r < 0.70:
            return int(self.succ[w2, np.searchsorted(self.succ_cdf, self.u())])
        return self.unigram()

    def sentence(self, markup: bool = False) -> str:
        n = 5 + int(self.u() * 21)
        w2, w1 = -1, -1
        toks = []
        for i in range(n):
            w = self.next_word(w2, w1)
            s = self.words[w]
            if i == 0:
                s = s.capitalize()
            if markup:
                r = self.u()
                if r < 0.10:
                    s = "[[" + s + "]]" if self.u() < 0.7 else "[[" + s + "|" + self.words[self.unigram()] + "]]"
                elif r < 0.12:
                    s = "'''" + s + "'''"
                elif r < 0.135:
                    s = s + "&lt;ref&gt;" + self.words[self.unigram()] + "&lt;/ref&gt;"
                elif r < 0.15:
                    s = str(int(self.u() * 2000) + 25)
                elif r < 0.165:
                    ch = NON_ASCII[int(self.u() * len(NON_ASCII))]
                    s = s[: len(s) // 2] + ch + s[len(s) // 2:]
            toks.append(s)
            if i < n - 1 and self.u() < 0.08:
                toks[-1] += ","
            if i < n - 1 and self.u() < 0.01:
                toks[-1] += ";"
            w2, w1 = w1, w
        end = "." if self.u() < 0.8 else ("!" if self.u() < 0.5 else "?")
        body = " ".join(toks) + end
        if not markup and self.u() < 0.2:
            tag = " said " + self.words[self.unigram()].capitalize() + "."
            body = '"' + body + '"' + tag
        return body


def _wrap(par: str, width: int = 72) -> str:
    lines, cur = [], ""
    for w in par.split(" "):
        if cur and len(cur) + 1 + len(w) > width:
            lines.append(cur)
            cur = w
        else:
            cur = w if not cur else cur + " " + w
    if cur:
        lines.append(cur)
    return "\n".join(lines)


def _roman(n: int) -> str:
    vals = [(1000, "M"), (900, "CM"), (500, "D"), (400, "CD"), (100, "C"), (90, "XC"),
            (50, "L"), (40, "XL"), (10, "X"), (9, "IX"), (5, "V"), (4, "IV"), (1, "I")]
    out = ""
    for v, s in vals:
        while n >= v:
            out += s
            n -= v
    return out


def _alice(n_bytes: int, seed: int) -> bytes:
    pr = _Prose(seed)
    parts, size, chapter, next_chapter = [], 0, 0, 0
    while size < n_bytes:
        if size >= next_chapter:
            chapter += 1
            title = " ".join(pr.words[pr.unigram()].capitalize() for _ in range(2 + int(pr.u() * 4)))
            s = "CHAPTER " + _roman(chapter) + ".\n" + title + "\n\n"
            next_chapter = size + 15000
        else:
            nsent = 2 + int(pr.u() * 6)
            s = _wrap(" ".join(pr.sentence() for _ in range(nsent))) + "\n\n"
        parts.append(s)
        size += len(s)
    return "".join(parts).encode("ascii")[:n_bytes]


def _enwik(n_bytes: int, seed: int) -> bytes:
    pr = _Prose(seed)
    out, size, page_id = [], 0, 0
    out.append('<mediawiki xmlns="http://www.mediawiki.org/xml/export-0.3/" version="0.3">\n')
    while size < n_bytes:
        page_id += 1
        title = " ".join(pr.words[pr.unigram()].capitalize() for _ in range(1 + int(pr.u() * 3)))
        body = []
        for sec in range(1 + int(pr.u() * 4)):
            if sec:
                body.append("== " + pr.words[pr.unigram()].capitalize() + " ==\n")
            if pr.u() < 0.3:
                body.append("{{" + pr.words[pr.unigram()] + "|" + pr.words[pr.unigram()] + "}}\n")
            body.append(" ".join(pr.sentence(markup=True) for _ in range(2 + int(pr.u() * 6))) + "\n")
            if pr.u() < 0.3:
                for _ in range(2 + int(pr.u() * 4)):
                    body.append("* [[" + pr.words[pr.unigram()] + "]]\n")
        year = 2001 + int(pr.u() * 6)
        page = ("  <page>\n    <title>" + title + "</title>\n    <id>" + str(page_id) + "</id>\n"
                "    <revision>\n      <id>" + str(100000 + page_id * 7) + "</id>\n"
                "      <timestamp>" + "%04d-%02d-%02dT%02d:%02d:%02dZ" % (
                    year, 1 + int(pr.u() * 12), 1 + int(pr.u() * 28), int(pr.u() * 24),
                    int(pr.u() * 60), int(pr.u() * 60)) + "</timestamp>\n"
                "      <text xml:space=\"preserve\">" + "".join(body)
                + "[[Category:" + pr.words[pr.unigram()].capitalize() + "]]</text>\n"
                "    </revision>\n  </page>\n")
        out.append(page)
        size += len(page.encode("utf-8"))
    data = "".join(out).encode("utf-8")[:n_bytes]
    return data


def _mixed(n_bytes: int, seed: int) -> bytes:
    """An arbitrary-file-shaped input for NC06: alice-shaped text segments
    (200 B - 6 KB) alternating with binary segments -- random bytes (incompressible),
    zero runs, small integer tables -- plus the cases the segmenter's rules act on:
    control-byte gaps of 1-12 bytes inside text, short printable runs (< 64 B) inside
    binary, and short binary chunks (< 64 B) next to text."""
    rng = np.random.default_rng(seed)
    prose = _alice(max(4 * n_bytes, 20000), seed + 1)
    out, pos = [], 0
    while sum(len(x) for x in out) < n_bytes:
        r = rng.random()
        if r < 0.45:                                       # text, maybe with small gaps
            ln = int(rng.integers(200, 6000))
            t = bytearray(prose[pos:pos + ln])
            pos = (pos + ln) % (len(prose) - 6000)
            for _ in range(int(rng.integers(0, 3))):
                at = int(rng.integers(0, max(1, len(t))))
                t[at:at] = bytes(rng.integers(0, 9, int(rng.integers(1, 13))).astype(np.uint8))
            out.append(bytes(t))
        elif r < 0.65:                                     # random bytes
            out.append(bytes(rng.integers(0, 256, int(rng.integers(16, 3000))).astype(np.uint8)))
        elif r < 0.8:                                      # zero runs / small tables
            n = int(rng.integers(8, 2000))
            out.append(bytes(n) if rng.random() < 0.5 else
                       np.arange(n // 4, dtype="<u4").tobytes())
        else:                                              # binary with short printable runs
            b = bytearray(rng.integers(128, 256, int(rng.integers(20, 400))).astype(np.uint8))
            at = int(rng.integers(0, len(b)))
            b[at:at] = b"header" + bytes(rng.integers(48, 58, int(rng.integers(1, 40))).astype(np.uint8))
            out.append(bytes(b))
    return b"".join(out)[:n_bytes]


def make_text(kind: str, n_bytes: int, seed: int) -> bytes:
    if kind == "alice":
        return _alice(n_bytes, seed)
    if kind == "enwik":
        return _enwik(n_bytes, seed)
    if kind == "mixed":
        return _mixed(n_bytes, seed)
    raise ValueError(kind)
