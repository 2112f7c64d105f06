"""Host-side mirror of the reference's tag-stream contract (input encoding of the hot path).

grammar::lex (grammar.cpp:51-89) splits text into the ten atomic tag literals and text
runs; tok::Tokenizer (tokenizer.cpp:24-101, Whitespace mode) gives tags the fixed ids
0..9 (TagKind order, grammar.hpp:34-46) and text words first-seen vocabulary ids from 10.
The device mask/position kernel consumes exactly these ids.
"""
from __future__ import annotations

TAGS = ("<Parallel>", "</Parallel>", "<Goal>", "</Goal>", "<Outline>", "</Outline>", "<Path>", "</Path>",
        "<Conclusion>", "</Conclusion>")
PAR_OPEN, PAR_CLOSE, GOAL_OPEN, GOAL_CLOSE, OUT_OPEN, OUT_CLOSE, PATH_OPEN, PATH_CLOSE, CONC_OPEN, CONC_CLOSE = range(10)
_WS = " \t\r\n"


def lex(source: str):
    """[(kind, raw)], kind = tag id or -1 for a text run (grammar.cpp:51-89)."""
    out, text_begin, i = [], 0, 0
    while i < len(source):
        if source[i] != "<":
            i += 1
            continue
        hit = next((k for k, lit in enumerate(TAGS) if source.startswith(lit, i)), None)
        if hit is None:
            i += 1
            continue
        if i > text_begin:
            out.append((-1, source[text_begin:i]))
        out.append((hit, TAGS[hit]))
        i += len(TAGS[hit])
        text_begin = i
    if len(source) > text_begin:
        out.append((-1, source[text_begin:]))
    return out


class Vocab:
    """Deterministic first-seen vocabulary with the tags pre-seeded at 0..9 (tokenizer.cpp:24-31)."""

    def __init__(self):
        self.entries = list(TAGS)
        self.index = {t: k for k, t in enumerate(TAGS)}

    def id_of(self, text: str) -> int:
        k = self.index.get(text)
        if k is None:
            k = len(self.entries)
            self.index[text] = k
            self.entries.append(text)
        return k


def tokenize(source: str, vocab: Vocab | None = None) -> list[int]:
    vocab = vocab or Vocab()
    ids = []
    for kind, raw in lex(source):
        if kind >= 0:
            ids.append(kind)
        else:
            word = ""
            for ch in raw + " ":
                if ch in _WS:
                    if word:
                        ids.append(vocab.id_of(word))
                        word = ""
                else:
                    word += ch
    return ids
