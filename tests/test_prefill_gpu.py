"""K3 parity: branch-masked prefill vs the fp64 oracle restatement of ToyModel::forward's
attention (toy_model.cpp:174-202: per row, visible rows in layout order, then self), GQA
h -> h/(Hq/Hkv), on bf16-rounded seeded inputs. Tolerance: max-abs 2e-3 (fp32 output)."""
import numpy as np
import pytest
import torch

import oracle
from mvtest import bf16_to_f64, record_margin, sym_bf16
from tools.workloads import nested_16k

pytestmark = pytest.mark.gpu
TOL = 2e-3


@pytest.fixture(scope="module")
def mv():
    import paper_2506_09991_b200 as m
    return m


def run_prefill(mv, tokens, hq, hkv, rows=None, seed=3, spike=None, d=128):
    """Device prefill (K1 intervals -> K3) against the oracle built from the tag stream alone: the oracle's
    own positions (dag.cpp:203-222 restated) and dense build_mask rows (dag.cpp:227-263), so a K1 bug cannot
    be certified by this test."""
    n = len(tokens)
    spec = mv.dag.build_visibility(tokens)
    q = sym_bf16(seed * 10 + 1, (n, hq, d))
    k = sym_bf16(seed * 10 + 2, (n, hkv, d))
    if spike is not None:
        # one key whose score dwarfs every other (dims 124-127 barely rotate: theta ~1e-4 rad per position)
        q[:, :, d - 4:] = 1.0
        k[spike, :, :] = 0.0
        k[spike, :, d - 4:] = 512.0
    v = sym_bf16(seed * 10 + 3, (n, hkv, d))
    out = mv.attention.prefill(q.cuda(), k.cuda(), v.cuda(), spec.positions, spec.excl, out_dtype=torch.float32)
    torch.cuda.synchronize()
    err_code, pos, _, _ = oracle.build_dag(tokens)
    assert err_code == 0
    rows = np.arange(n) if rows is None else np.asarray(rows)
    Kr = oracle.rope(bf16_to_f64(k), pos)
    qr = oracle.rope(bf16_to_f64(q)[rows], pos[rows])
    ref = oracle.attn_prefill_tokens(qr, Kr, bf16_to_f64(v), tokens, rows)
    got = out.cpu().numpy()[rows]
    err = float(np.abs(got - ref).max())
    tag = f"prefill n={n} hq={hq}/{hkv} rows={len(rows)}" + (f" d={d}" if d != 128 else "")
    record_margin(tag, err, TOL)
    if n <= 5000:
        # where the error comes from: the kernels hold rotated Q and K in bf16 (MMA operands, as a bf16 KV
        # cache does); the same oracle on bf16-rounded rotated q / k leaves only the bf16 P rounding
        r16 = lambda a: torch.from_numpy(a).to(torch.bfloat16).double().numpy()  # noqa: E731
        ref16 = oracle.attn_prefill_tokens(r16(qr), r16(Kr), bf16_to_f64(v), tokens, rows)
        record_margin(tag + " vs oracle(bf16 rotated q/k)", float(np.abs(got - ref16).max()), TOL)
    return err, spec


def test_t1_all_rows(mv, dag_golden):
    t1 = next(c for c in dag_golden if c["name"] == "fixture:t1.txt")
    err, _ = run_prefill(mv, t1["tokens"], hq=8, hkv=2)
    assert err < TOL, err


@pytest.mark.parametrize("spike", [142, 174, 190, 206])
def test_score_spike(mv, dag_golden, spike):
    """A key ~260 log2 units above every other score, in a later key tile than the row's first: the
    softmax reference must move (sum guard) even when the key sits on a polynomial-exp2 column
    (key % 64 in {14, 15, 30, 31, 46, 47, 62, 63}); rows that see it return its value row exactly."""
    nested = next(c for c in dag_golden if c["name"] == "fixture:nested.txt")
    err, _ = run_prefill(mv, nested["tokens"], hq=8, hkv=2, spike=spike)
    assert err < TOL, err


def test_random_trajectories(mv, dag_golden):
    cases = [c for c in dag_golden if c["name"].startswith("random4x6") and c["error"] == -1][:6]
    for c in cases:
        err, _ = run_prefill(mv, c["tokens"], hq=40, hkv=8, seed=len(c["tokens"]))
        assert err < TOL, (c["name"], err)


def test_nested_fixture_known_positions(mv, dag_golden):
    nested = next(c for c in dag_golden if c["name"] == "fixture:nested.txt")
    err, spec = run_prefill(mv, nested["tokens"], hq=40, hkv=8)
    assert err < TOL, err
    assert spec.positions.cpu().tolist() == nested["positions"]


def test_c3_nested_16k_sampled(mv):
    # BASELINE configs[2]: 16K structured sequence, nested Parallel blocks, Qwen head shape
    toks = nested_16k()
    rng = np.random.default_rng(0)
    rows = np.sort(np.concatenate([rng.choice(16384, 60, replace=False), [0, 1, 16383, 2048, 2049]]))
    err, spec = run_prefill(mv, toks, hq=40, hkv=8, rows=rows)
    assert err < TOL, err


def nested_tokens(depth, paths, path_words, seed=0, prefix=100):
    """A tag stream with Parallel blocks nested `depth` deep (every path of a block holds another
    block until the innermost level): many exclusion intervals per row, interval ends inside k
    tiles, and short sibling paths that share a 128-token tile."""
    rng = np.random.default_rng(seed)
    words = lambda k: [int(x) for x in 10 + rng.integers(0, 4000, size=k)]  # noqa: E731
    P_OPEN, P_CLOSE, G_OPEN, G_CLOSE, O_OPEN, O_CLOSE, PATH, PATH_C, C_OPEN, C_CLOSE = range(10)

    def block(d):
        t = [P_OPEN, G_OPEN]
        for _ in range(paths):
            t += [O_OPEN] + words(3) + [O_CLOSE]
        t += [G_CLOSE]
        for _ in range(paths):
            body = words(path_words)
            if d > 1:
                body += block(d - 1) + words(max(1, path_words // 2))
            t += [PATH] + body + [PATH_C]
        return t + [C_OPEN] + words(5) + [C_CLOSE, P_CLOSE]

    return words(prefix) + block(depth) + words(7)


@pytest.mark.parametrize("depth,paths,pw", [(3, 3, 20), (4, 2, 9), (2, 6, 5)])
def test_deep_nesting_all_rows(mv, depth, paths, pw):
    toks = nested_tokens(depth, paths, pw, seed=depth * 10 + paths)
    err, spec = run_prefill(mv, toks, hq=40, hkv=8, seed=depth)
    assert spec.excl.shape[1] >= depth - 1
    assert err < TOL, (len(toks), err)


@pytest.mark.parametrize("hq,hkv", [(4, 4), (16, 2), (8, 8), (1, 1)])
def test_gqa_ratios(mv, dag_golden, hq, hkv):
    c = next(c for c in dag_golden if c["name"].startswith("random4x6") and c["error"] == -1)
    err, _ = run_prefill(mv, c["tokens"], hq=hq, hkv=hkv, seed=hq + hkv)
    assert err < TOL, err


def test_bf16_output_matches_fp32(mv):
    toks = nested_tokens(3, 3, 40, seed=7)
    n = len(toks)
    spec = mv.dag.build_visibility(toks)
    q, k, v = sym_bf16(71, (n, 40, 128)).cuda(), sym_bf16(72, (n, 8, 128)).cuda(), sym_bf16(73, (n, 8, 128)).cuda()
    o32 = mv.attention.prefill(q, k, v, spec.positions, spec.excl, out_dtype=torch.float32)
    o16 = mv.attention.prefill(q, k, v, spec.positions, spec.excl)
    # identical arithmetic, then the bf16 store rounding (<= 2^-9 relative)
    d = (o16.float() - o32).abs()
    assert bool((d <= o32.abs() * 2.0 ** -8 + 1e-6).all())


def test_sequence_lengths_around_tiles(mv):
    # lengths that leave a partial last q tile / k tile, including n < 128 and n = 128 * k + 1
    for n_extra in (0, 1, 127, 129, 255, 383):
        toks = nested_tokens(2, 2, 8, seed=n_extra, prefix=50 + n_extra)
        err, spec = run_prefill(mv, toks, hq=8, hkv=2, seed=n_extra + 1)
        assert err < TOL, (len(toks), err)
        # the bf16 output leaves through a TMA store of whole 128-row tiles: rows past n are clipped,
        # rows before it equal the fp32 result up to the bf16 rounding
        n = len(toks)
        q, k, v = sym_bf16(n + 1, (n, 8, 128)).cuda(), sym_bf16(n + 2, (n, 2, 128)).cuda(), sym_bf16(n + 3, (n, 2, 128)).cuda()
        guard = torch.full((n + 256, 8, 128), 7.0, dtype=torch.bfloat16, device="cuda")
        o16 = guard[:n]
        mv.attention.prefill(q, k, v, spec.positions, spec.excl, out=o16)
        o32 = mv.attention.prefill(q, k, v, spec.positions, spec.excl, out_dtype=torch.float32)
        d = (o16.float() - o32).abs()
        assert bool((d <= o32.abs() * 2.0 ** -8 + 1e-6).all()), n
        assert bool((guard[n:] == 7.0).all()), n  # nothing written past row n


def test_32k_nested_sampled(mv):
    """A ~33K-token stream (twice configs[2]; two top-level blocks, three nesting levels): tile
    lists, the RoPE table and the persistent queue beyond the benchmark size; sampled rows
    against the oracle."""
    toks = nested_tokens(3, 4, 290, seed=32, prefix=2000) + nested_tokens(2, 3, 300, seed=33, prefix=100)
    rng = np.random.default_rng(3)
    n = len(toks)
    assert 30000 < n < 40000, n
    rows = np.sort(np.concatenate([rng.choice(n, 48, replace=False), [0, n - 1]]))
    err, spec = run_prefill(mv, toks, hq=40, hkv=8, rows=rows, seed=9)
    assert err < TOL, (n, err)


def deep_chain(depth, seed=0):
    """A tag stream nested `depth` blocks deep along one path per level (linear size): every row of the
    innermost path carries `depth` exclusion intervals (the reference's recursion has no limit,
    dag.cpp:117-187)."""
    rng = np.random.default_rng(seed)
    words = lambda k: [int(x) for x in 10 + rng.integers(0, 4000, size=k)]  # noqa: E731
    P_OPEN, P_CLOSE, G_OPEN, G_CLOSE, O_OPEN, O_CLOSE, PATH, PATH_C, C_OPEN, C_CLOSE = range(10)

    def block(d):
        t = [P_OPEN, G_OPEN, O_OPEN] + words(2) + [O_CLOSE, O_OPEN] + words(2) + [O_CLOSE, G_CLOSE]
        t += [PATH] + words(6) + [PATH_C]
        t += [PATH] + words(5) + (block(d - 1) if d > 1 else []) + words(3) + [PATH_C]
        return t + [C_OPEN] + words(3) + [C_CLOSE, P_CLOSE]

    return words(40) + block(depth) + words(9)


def test_nesting_deeper_than_eight(mv):
    """12 nested blocks: K1 grows its interval capacity, the tile map and K3 read the intervals beyond 8
    from memory; every row against the oracle's own mask."""
    toks = deep_chain(12)
    err, spec = run_prefill(mv, toks, hq=8, hkv=2, seed=12)
    assert spec.excl.shape[1] >= 12
    assert err < TOL, err


# ---- head dim 64 (the toy model's d_h, toy_model.hpp:29): native prefill_tc3_kernel<64> ----
def test_head_dim_64_t1_and_trajectories(mv, dag_golden):
    t1 = next(c for c in dag_golden if c["name"] == "fixture:t1.txt")["tokens"]
    err, _ = run_prefill(mv, t1, 4, 4, d=64)
    assert err < TOL, err
    for c in [c for c in dag_golden if c["name"].startswith("random4x6") and c["error"] == -1][:6]:
        err, _ = run_prefill(mv, c["tokens"], 40, 8, d=64, seed=len(c["tokens"]))
        assert err < TOL, (c["name"], err)


@pytest.mark.parametrize("depth,paths,pw", [(2, 3, 40), (3, 2, 60)])
def test_head_dim_64_nested(mv, depth, paths, pw):
    err, _ = run_prefill(mv, nested_tokens(depth, paths, pw, seed=depth), 40, 8, d=64)
    assert err < TOL


def test_head_dim_64_spike_and_tiles(mv, dag_golden):
    toks = nested_tokens(2, 3, 40, seed=9)
    err, _ = run_prefill(mv, toks, 8, 2, spike=len(toks) // 2, d=64)
    assert err < TOL
    for n in (1, 127, 129, 300):
        err, _ = run_prefill(mv, list(range(30, 30 + n)), 8, 2, d=64, seed=n)
        assert err < TOL


def test_head_dim_64_bf16_output(mv):
    toks = nested_tokens(2, 3, 40, seed=13)
    n = len(toks)
    spec = mv.dag.build_visibility(toks)
    q, k, v = sym_bf16(81, (n, 8, 64)).cuda(), sym_bf16(82, (n, 2, 64)).cuda(), sym_bf16(83, (n, 2, 64)).cuda()
    o32 = mv.attention.prefill(q, k, v, spec.positions, spec.excl, out_dtype=torch.float32)
    o16 = mv.attention.prefill(q, k, v, spec.positions, spec.excl)
    d = (o16.float() - o32).abs()
    assert bool((d <= o32.abs() * 2.0 ** -8 + 1e-6).all())
