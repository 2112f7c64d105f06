"""Layout edits on tag streams (host-side, token ids): the SPEC's permutation / isolation
properties (AC-4, AC-5) as inputs for the GPU prefill.

`permute_paths` restates multiverse::dag::permute_paths (dag.cpp:272-306) on the token stream
instead of the GenerationDag layout: the tokens of every path subtree of block `block_index`
(a `<Path>` ... `</Path>` span, nested blocks included) form the region; the region's slots are
refilled, in layout order, with the subtrees in the order `perm` names. Blocks are numbered in
the order their `<Parallel>` opens, as build_dag creates them (DFS, dag.cpp:117-119).
"""
from __future__ import annotations

from .tokenize import PAR_CLOSE, PAR_OPEN, PATH_CLOSE, PATH_OPEN


def blocks(tokens) -> list[list[tuple[int, int]]]:
    """Per block (opening order): the [begin, end) token span of each of its paths, `<Path>` and
    `</Path>` included. Raises ValueError on unbalanced tags (grammar::ParseError's job upstream)."""
    out: list[list[tuple[int, int]]] = []
    stack: list[int] = []      # open blocks (indices into out)
    path_open: list[int] = []  # start of the open path of each stacked block (-1: none)
    for i, t in enumerate(int(x) for x in tokens):
        if t == PAR_OPEN:
            stack.append(len(out))
            out.append([])
            path_open.append(-1)
        elif t == PAR_CLOSE:
            if not stack or path_open[-1] != -1:
                raise ValueError(f"unbalanced </Parallel> at {i}")
            stack.pop()
            path_open.pop()
        elif t == PATH_OPEN:
            if not stack or path_open[-1] != -1:
                raise ValueError(f"<Path> outside a block at {i}")
            path_open[-1] = i
        elif t == PATH_CLOSE:
            if not stack or path_open[-1] == -1:
                raise ValueError(f"unbalanced </Path> at {i}")
            out[stack[-1]].append((path_open[-1], i + 1))
            path_open[-1] = -1
    if stack:
        raise ValueError("unclosed <Parallel>")
    return out


def permute_paths(tokens, block_index: int, perm) -> list[int]:
    """dag::permute_paths (dag.cpp:272-306) on token ids; same errors: std::out_of_range for a bad
    block index (IndexError here), std::invalid_argument when perm's size is not the path count."""
    toks = [int(x) for x in tokens]
    return [toks[s] for s in permutation_source(toks, block_index, perm)]


def permutation_source(tokens, block_index: int, perm) -> list[int]:
    """src with permute_paths(tokens, b, perm)[i] == tokens[src[i]] (the row map the parity tests
    compare outputs through)."""
    toks = [int(x) for x in tokens]
    spans = blocks(toks)[block_index]
    perm = [int(p) for p in perm]
    if len(perm) != len(spans):
        raise ValueError("permutation size does not match path count")
    if sorted(perm) != list(range(len(spans))):
        raise ValueError("not a permutation")
    region = [i for b, e in spans for i in range(b, e)]   # region_slots (dag.cpp:286-297)
    fill = [i for p in perm for i in range(*spans[p])]
    src = list(range(len(toks)))
    for slot, i in zip(region, fill):
        src[slot] = i
    return src


def path_rows(tokens, block_index: int, path: int) -> range:
    """Token rows of one path subtree of a block."""
    return range(*blocks(tokens)[block_index][path])
