"""K1 parity: the device mask/position builder against the patched reference's goldens
(tests/golden/dag.jsonl.gz) and the CPU oracle, bit-exact."""
import numpy as np

from tools.workloads import nested_16k  # noqa: F401  (also imported by test_prefill_gpu)
import pytest
import torch

import oracle
from conftest import fnv1a

pytestmark = pytest.mark.gpu

REF_ERR = {-1: 0, 0: 5, 1: 6}  # ParseError::Kind -> mv_status


@pytest.fixture(scope="module")
def mv():
    import paper_2506_09991_b200 as m
    return m


def test_goldens_batched_one_launch(mv, dag_golden):
    specs, status = mv.dag.build_visibility_batch([c["tokens"] for c in dag_golden], max_depth=6)
    n_ok = 0
    for case, spec, st in zip(dag_golden, specs, status):
        assert st == REF_ERR[case["error"]], case["name"]
        if st:
            continue
        n_ok += 1
        assert spec.positions.cpu().tolist() == case["positions"], case["name"]
        assert spec.seg_id.cpu().tolist() == case["seg"], case["name"]
        packed = spec.mask_packed().cpu().numpy()
        assert fnv1a(packed.tobytes()) == case["mask_fnv"], case["name"]
        if "mask_hex" in case:
            assert packed.tobytes().hex() == case["mask_hex"], case["name"]
    assert n_ok > 300


def test_t1_single(mv, dag_golden):
    t1 = next(c for c in dag_golden if c["name"] == "fixture:t1.txt")
    spec = mv.dag.build_visibility(t1["tokens"])
    m = spec.mask().cpu().numpy()
    assert not m[17:23, 12:17].any() and m[23, :23].all()
    assert spec.positions.cpu().tolist()[12:23] == [12, 13, 14, 15, 16, 12, 13, 14, 15, 16, 17]


def test_parse_errors_raise(mv):
    with pytest.raises(mv.ParseError) as e:
        mv.dag.build_visibility([0, 2, 3])  # <Parallel><Goal></Goal>: zero outlines
    assert e.value.kind == "CountMismatch"
    with pytest.raises(mv.ParseError) as e:
        mv.dag.build_visibility([6, 10])  # <Path> at top level
    assert e.value.kind == "MalformedStructure"


def test_edge_cases(mv):
    # empty stream, text only, a block at position 0, depth capacity
    specs, st = mv.dag.build_visibility_batch([[], [10, 11, 12], [0, 2, 4, 5, 3, 6, 7, 8, 9, 1]], max_depth=1)
    assert st == [0, 0, 0]
    assert specs[1].positions.cpu().tolist() == [0, 1, 2]
    assert specs[2].positions.cpu().tolist() == list(range(10))


def test_nested_16k_against_oracle(mv):
    toks = nested_16k()
    assert len(toks) == 16384
    err, pos, seg, _ = oracle.build_dag(toks)
    assert err == 0
    spec = mv.dag.build_visibility(toks)
    assert np.array_equal(spec.positions.cpu().numpy(), pos)
    assert np.array_equal(spec.seg_id.cpu().numpy(), seg)
    n = len(toks)
    for r0 in range(0, n, 2048):  # dense mask in row blocks (the oracle streams rows too)
        r1 = min(n, r0 + 2048)
        ref = oracle.mask_packed(toks, r0, r1)
        got = spec.mask_packed(r0, r1).cpu().numpy()
        assert np.array_equal(got, ref), (r0, r1)


def test_tile_map_counts_visible_pairs(mv):
    toks = nested_16k()
    spec = mv.dag.build_visibility(toks)
    count, lst, vis = mv.dag.tile_map(spec, 128)
    n = len(toks)
    total = 0
    for r0 in range(0, n, 4096):
        total += int(np.unpackbits(oracle.mask_packed(toks, r0, min(n, r0 + 4096))).sum())
    assert int(vis.item()) == total
    # every visible pair lies in a listed tile; skipped tiles hold no visible pair
    dense_rows = np.unpackbits(oracle.mask_packed(toks, 0, 1024))[: 1024 * n].reshape(1024, n)
    c = count.cpu().numpy()
    L = lst.cpu().numpy()
    for qt in range(1024 // 128):
        listed = {int(x) & 0xFFFF for x in L[qt, : c[qt]]}
        for kt in range(qt + 1):
            blk = dense_rows[qt * 128:(qt + 1) * 128, kt * 128:(kt + 1) * 128]
            assert (kt in listed) == bool(blk.any())


def test_training_batch_targets_match_reference(mv):
    """§8f-4: the device training batch (targets, loss masks with / without tag loss, positions) equals
    the reference's build_training_batch on every parse-valid golden trajectory (tests/golden/batch.jsonl.gz)."""
    from conftest import load_jsonl
    rows = load_jsonl("batch.jsonl.gz")
    for r in rows:
        b = mv.dag.build_training_batch(r["tokens"], tag_loss=True, max_depth=8)
        assert b.target_ids.cpu().tolist() == r["targets"], r["name"]
        assert b.loss_mask.cpu().tolist() == r["loss_mask"], r["name"]
        b2 = mv.dag.build_training_batch(r["tokens"], tag_loss=False, max_depth=8)
        assert b2.loss_mask.cpu().tolist() == r["loss_mask_no_tags"], r["name"]
        err, pos, _, _ = oracle.build_dag(r["tokens"])
        assert b.positions.cpu().tolist() == pos.tolist(), r["name"]


def test_training_batch_16k_against_oracle(mv):
    toks = nested_16k()
    b = mv.dag.build_training_batch(toks, tag_loss=False)
    err, tgt, loss = oracle.batch_targets(toks, False)
    assert err == 0
    assert np.array_equal(b.target_ids.cpu().numpy(), tgt) and np.array_equal(b.loss_mask.cpu().numpy(), loss)
