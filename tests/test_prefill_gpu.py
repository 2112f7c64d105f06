"""K3 parity: branch-masked prefill vs the fp64 oracle restatement of ToyModel::forward's
attention (toy_model.cpp:174-202: per row, visible rows in layout order, then self), GQA
h -> h/(Hq/Hkv), on bf16-rounded seeded inputs. Tolerance: max-abs 2e-3 (fp32 output)."""
import numpy as np
import pytest
import torch

import oracle
from mvtest import bf16_to_f64, sym_bf16
from test_visibility_gpu import nested_16k

pytestmark = pytest.mark.gpu
TOL = 2e-3


@pytest.fixture(scope="module")
def mv():
    import paper_2506_09991_b200 as m
    return m


def run_prefill(mv, tokens, hq, hkv, rows=None, seed=3):
    n = len(tokens)
    spec = mv.dag.build_visibility(tokens)
    q = sym_bf16(seed * 10 + 1, (n, hq, 128))
    k = sym_bf16(seed * 10 + 2, (n, hkv, 128))
    v = sym_bf16(seed * 10 + 3, (n, hkv, 128))
    out = mv.attention.prefill(q.cuda(), k.cuda(), v.cuda(), spec.positions, spec.excl, out_dtype=torch.float32)
    torch.cuda.synchronize()
    pos = spec.positions.cpu().numpy()
    rows = np.arange(n) if rows is None else np.asarray(rows)
    Kr = oracle.rope(bf16_to_f64(k), pos)
    qr = oracle.rope(bf16_to_f64(q)[rows], pos[rows])
    ref = oracle.attn_prefill(qr, Kr, bf16_to_f64(v), spec.excl.cpu().numpy(), rows)
    got = out.cpu().numpy()[rows]
    return float(np.abs(got - ref).max()), spec


def test_t1_all_rows(mv, dag_golden):
    t1 = next(c for c in dag_golden if c["name"] == "fixture:t1.txt")
    err, _ = run_prefill(mv, t1["tokens"], hq=8, hkv=2)
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
