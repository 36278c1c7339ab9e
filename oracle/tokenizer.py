"""Tokenizer over the synthetic vocabulary (SURVEY.md D30 reading of P:305-311).

The paper tokenizes with SmolLM2's HF BPE, unavailable offline.  Our
reading: greedy longest match over the model vocabulary, specials (ids <
n_special) never matched; every byte is a token, so tokenize is total and
detokenize(tokenize(x)) == x (the round-trip contract).  A string present under
several ids maps to the LOWEST id (D30; pinned by
test_tokenizer_duplicate_string_lowest_id_wins).
"""


class Tokenizer:
    def __init__(self, vocab, n_special=3):
        self.vocab = list(vocab)
        self.n_special = n_special
        self.lookup = {}
        for i, s in enumerate(self.vocab):
            if i >= n_special and s not in self.lookup:   # lowest id wins (D30)
                self.lookup[s] = i
        self.max_len = max(len(s) for s in self.vocab[n_special:])

    def encode(self, data: bytes):
        out, i, n = [], 0, len(data)
        lookup, max_len = self.lookup, self.max_len
        while i < n:
            for ln in range(min(max_len, n - i), 0, -1):
                tid = lookup.get(data[i:i + ln])
                if tid is not None:
                    out.append(tid)
                    i += ln
                    break
            else:  # unreachable: every single byte is in the vocabulary
                raise ValueError("byte not in vocabulary")
        return out

    def decode(self, ids) -> bytes:
        return b"".join(self.vocab[i] for i in ids)
