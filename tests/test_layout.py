"""Host-side layout edits (paper_2506_09991_b200/host/layout.py) pinned by the CPU oracle.

permute_paths restates dag::permute_paths (dag.cpp:272-306) on token ids. SPEC.md:180-181
states why positions and mask are layout-order-invariant under it; here that is checked
exactly on the reference-generated golden trajectories: the permuted stream parses, and its
positions and dense mask equal the original's taken through the row map. No GPU needed."""
import itertools

import numpy as np
import pytest

import oracle
from paper_2506_09991_b200.host import layout
from paper_2506_09991_b200.host.tokenize import tokenize

NESTED = ("intro words here <Parallel> <Goal> <Outline> 1: a </Outline> <Outline> 2: b </Outline> "
          "<Outline> 3: c </Outline> </Goal> <Path> 1: x x <Parallel> <Goal> <Outline> 1: u </Outline> "
          "<Outline> 2: v </Outline> </Goal> <Path> 1: p q r </Path> <Path> 2: s t </Path> <Conclusion> w "
          "</Conclusion> </Parallel> y </Path> <Path> 2: z z z z </Path> <Path> 3: k </Path> <Conclusion> "
          "done now </Conclusion> </Parallel> tail")


def check_invariance(toks, b, perm):
    src = np.array(layout.permutation_source(toks, b, perm))
    new = layout.permute_paths(toks, b, perm)
    assert new == [toks[s] for s in src]
    assert sorted(src.tolist()) == list(range(len(toks)))
    e0, p0, _, _ = oracle.build_dag(toks)
    e1, p1, _, _ = oracle.build_dag(new)
    assert e0 == 0 and e1 == 0
    assert (p1 == p0[src]).all()
    m0, m1 = oracle.mask_dense(toks), oracle.mask_dense(new)
    assert (m1 == m0[np.ix_(src, src)]).all()
    return new, src


def test_nested_all_permutations():
    toks = tokenize(NESTED)
    spans = layout.blocks(toks)
    assert [len(s) for s in spans] == [3, 2]  # outer block 3 paths, inner (inside path 1) 2
    for b, s in enumerate(spans):
        for perm in itertools.permutations(range(len(s))):
            new, _ = check_invariance(toks, b, perm)
            inv = np.argsort(perm).tolist()
            assert layout.permute_paths(new, b, inv) == toks  # the inverse permutation restores the layout
    assert layout.permute_paths(toks, 0, [0, 1, 2]) == toks


def test_golden_trajectories_random_permutations(dag_golden):
    rng = np.random.default_rng(5)
    n_checked = 0
    for c in dag_golden:
        if c["error"] != -1 or len(c["tokens"]) > 400:
            continue
        spans = layout.blocks(c["tokens"])
        for b, s in enumerate(spans):
            if len(s) < 2:
                continue
            check_invariance(list(c["tokens"]), b, rng.permutation(len(s)).tolist())
            n_checked += 1
        if n_checked >= 60:
            break
    assert n_checked >= 30


def test_errors():
    toks = tokenize(NESTED)
    with pytest.raises(ValueError):
        layout.permute_paths(toks, 0, [0, 1])       # size mismatch (dag.cpp:275-277)
    with pytest.raises(ValueError):
        layout.permute_paths(toks, 0, [0, 0, 1])    # not a permutation
    with pytest.raises(IndexError):
        layout.permute_paths(toks, 2, [0])          # no such block (blocks.at)
    with pytest.raises(ValueError):
        layout.blocks(toks[:-3])                    # unclosed block


def toy_ref(toy_golden):
    c = toy_golden["t1_c1"]
    return oracle.Toy(c["layers"], c["heads"], c["model_dim"], c["vocab"], c["seed"], c["init"], c["rope"])


def ref_forward(ref, toks):
    err, pos, _, _ = oracle.build_dag(toks)
    assert err == 0
    return ref.forward(toks, pos, oracle.mask_dense(toks))


def test_oracle_toy_permutation_and_isolation(toy_golden):
    """AC-5 / AC-4 on the fp64 restatement: what the GPU property tests in
    test_properties_gpu.py hold the kernels to."""
    ref = toy_ref(toy_golden)
    toks = tokenize(NESTED)
    base = ref_forward(ref, toks)
    mask = oracle.mask_dense(toks)
    for b, spans in enumerate(layout.blocks(toks)):
        for perm in itertools.permutations(range(len(spans))):
            src = np.array(layout.permutation_source(toks, b, perm))
            got = ref_forward(ref, layout.permute_paths(toks, b, perm))
            assert np.abs(got - base[src]).max() <= 1e-5, (b, perm)
        for p in range(len(spans)):
            rows = np.arange(*spans[p])
            seen = mask[rows].any(0)
            seen[rows] = True
            new = [t if (seen[i] or t < 10) else t + 1 for i, t in enumerate(toks)]
            got = ref_forward(ref, new)
            assert np.abs(got[rows] - base[rows]).max() <= 1e-6, (b, p)
            assert np.abs(got - base).max() > 0  # the edit is visible somewhere
