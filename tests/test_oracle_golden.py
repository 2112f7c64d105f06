"""Pins the CPU oracle (oracle/mv_oracle.c) against the patched reference's own outputs.

Goldens were produced by oracle/refdrv.cpp linked against the reference core with the
two SURVEY.md §0 fixes (tests/golden/gen_golden.py). No GPU needed.
"""
import numpy as np
import pytest

import oracle
from conftest import fnv1a, kv_logs, load_jsonl

REF_ERR = {-1: 0, 0: 1, 1: 2}  # ParseError::Kind (grammar.hpp:138) -> oracle error code


def test_dag_goldens(dag_golden):
    n_ok = n_err = 0
    for case in dag_golden:
        err, pos, seg, kind = oracle.build_dag(case["tokens"])
        assert err == REF_ERR[case["error"]], case["name"]
        if err:
            n_err += 1
            continue
        n_ok += 1
        assert pos.tolist() == case["positions"], case["name"]
        assert seg.tolist() == case["seg"], case["name"]
        assert kind.tolist() == case["segkind"], case["name"]
        packed = oracle.mask_packed(case["tokens"])
        assert fnv1a(packed.tobytes()) == case["mask_fnv"], case["name"]
        if "mask_hex" in case:
            assert packed.tobytes().hex() == case["mask_hex"], case["name"]
    assert n_ok > 300 and n_err > 100


def test_t1_known_answers(dag_golden):
    t1 = next(c for c in dag_golden if c["name"] == "fixture:t1.txt")
    assert len(t1["tokens"]) == 28
    assert t1["positions"] == list(range(12)) + list(range(12, 17)) + list(range(12, 18)) + list(range(18, 23))
    m = oracle.mask_dense(t1["tokens"])
    assert not m[17:23, 12:17].any()  # path 2 never sees path 1
    assert m[23, :23].all()  # "done" sees all 23 prior tokens


def test_nested_known_answers(dag_golden):
    nested = next(c for c in dag_golden if c["name"] == "fixture:nested.txt")
    assert len(nested["tokens"]) == 218 and max(nested["seg"]) + 1 == 11


def test_toy_step_bit_exact(toy_golden):
    for name in ("step_small", "step_c1", "step_c1_empty"):
        g = toy_golden[name]
        toy = oracle.Toy(g["layers"], g["heads"], g["model_dim"], g["vocab"], g["seed"], g["init"], g["rope"])
        ctx = oracle.fill_symmetric(g["ctx_seed"], 1.0, g["ctx_len"] * toy.rec)
        logits, _, kv = toy.step(ctx, g["token"], g["pos"])
        np.testing.assert_array_equal(logits, np.array(g["logits"]))
        np.testing.assert_array_equal(kv, np.array(g["kv"]))


def test_toy_forward_bit_exact(toy_golden):
    for name in ("t1_small", "t1_c1"):
        g = toy_golden[name]
        toy = oracle.Toy(g["layers"], g["heads"], g["model_dim"], g["vocab"], g["seed"], g["init"], g["rope"])
        mask = oracle.mask_dense(g["tokens"])
        logits = toy.forward(g["tokens"], g["positions"], mask)
        np.testing.assert_array_equal(logits.reshape(-1), np.array(g["logits"]))


def test_forced_engine_equals_batch_forward(toy_golden):
    # engine::run_forced logits (KV through the radix store) == masked batch forward, bit-exact
    # (SURVEY.md §0 BUG-2 note); the oracle reproduces both from the token stream alone.
    for name, cfg in (("forced_t1_small", "t1_small"), ("forced_c1_mini", "t1_c1")):
        g = toy_golden[name]
        c = toy_golden[cfg]
        assert g["status"] == 0 and g["max_merge_bytes"] == 0
        toy = oracle.Toy(c["layers"], c["heads"], c["model_dim"], c["vocab"], c["seed"], c["init"], c["rope"])
        from paper_2506_09991_b200.host.tokenize import tokenize  # host mirror of tok::Tokenizer
        ids = tokenize(g["text"])
        err, pos, _, _ = oracle.build_dag(ids)
        assert err == 0
        logits = toy.forward(ids, pos, oracle.mask_dense(ids))
        np.testing.assert_array_equal(logits.reshape(-1), np.array(g["logits"]))


class FlatMirror:
    """tests/oracles.hpp:141-186, plus the RadixStore error contract (kvcache.cpp:16-20, 262-275).

    `slots` models physical sharing by lineage (fresh slot per appended token; fork/merge
    copy slot lists), which is the merge-descendant rule of a store without radix dedup.
    """

    def __init__(self):
        self.seq, self.slots = {}, {}
        self.next_id = 1
        self.fresh = 0

    def new(self, s, slots):
        h = self.next_id
        self.next_id += 1
        self.seq[h] = s
        self.slots[h] = slots
        return h

    def fresh_slots(self, k):
        self.fresh += k
        return list(range(self.fresh - k, self.fresh))


@pytest.mark.parametrize("log", kv_logs())
def test_kv_log_flat_mirror(log):
    rows = load_jsonl(log)
    m = FlatMirror()
    released = set()
    for r in rows[1:-1]:
        op, args = r["op"], r["args"]
        err, res = -1, []
        if op == "create":
            res = [m.new([], [])]
        elif op == "extend":
            res = [m.new(m.seq[args[0]] + r["tokens"], m.slots[args[0]] + m.fresh_slots(len(r["tokens"])))]
        elif op == "fork":
            res = [m.new(list(m.seq[args[0]]), list(m.slots[args[0]])) for _ in range(r["n"])]
        elif op == "merge":
            p, ps = m.seq[args[0]], m.slots[args[0]]
            ok = all(len(m.seq[b]) >= len(p) and m.slots[b][: len(p)] == ps for b in args[1:])
            if ok:
                s, sl = list(p), list(ps)
                for b in args[1:]:
                    s += m.seq[b][len(p):]
                    sl += m.slots[b][len(p):]
                res = [m.new(s, sl)]
            else:
                err = 3
        elif op == "release":
            if args[0] in m.seq:
                del m.seq[args[0]]
                released.add(args[0])
            else:
                err = 1
        assert err == r["error"], (log, r)
        assert res == r["results"], (log, r)
        assert sum(len(s) for s in m.seq.values()) == r["logical"]
        assert len(m.seq) == r["live"] and r["bytes_copied"] == 0
        for rv in r["resolved"]:
            assert m.seq[rv["id"]] == rv["tokens"]
    for rv in rows[-1]["final"]:
        assert m.seq[rv["id"]] == rv["tokens"]


def test_prefill_oracle_from_tokens_matches_dense_rule():
    """oracle.attn_prefill_tokens (mask from the oracle's build_mask rows, no intervals) equals a direct
    numpy evaluation of ToyModel::forward's attention (toy_model.cpp:183-196) over the dense mask."""
    import oracle
    t1 = [10, 0, 2, 4, 11, 12, 5, 4, 13, 14, 5, 3, 6, 11, 15, 16, 7, 6, 13, 17, 18, 19, 7, 8, 20, 9, 1, 21]
    n = len(t1)
    rng = np.random.default_rng(0)
    q, K, V = rng.uniform(-1, 1, (n, 4, 16)), rng.uniform(-1, 1, (n, 2, 16)), rng.uniform(-1, 1, (n, 2, 16))
    rows = np.array([0, 5, 12, 16, 17, 22, 23, 27])
    out = oracle.attn_prefill_tokens(q[rows], K, V, t1, rows)
    M = oracle.mask_dense(t1)
    for r, i in enumerate(rows):
        ctx = [j for j in range(i) if M[i, j]] + [i]
        for h in range(4):
            s = np.array([q[i, h] @ K[j, h // 2] for j in ctx]) / 4.0
            p = np.exp(s - s.max())
            assert np.abs(out[r, h] - (p[:, None] * V[ctx, h // 2]).sum(0) / p.sum()).max() < 1e-12


def test_batch_targets_oracle_matches_reference():
    """The oracle's build_training_batch restatement equals the reference's targets and loss masks
    (tests/golden/batch.jsonl.gz: refdrv batch over every parse-valid dag-golden trajectory)."""
    import oracle
    rows = load_jsonl("batch.jsonl.gz")
    assert len(rows) > 300
    for r in rows:
        err, tgt, loss = oracle.batch_targets(r["tokens"], True)
        assert err == 0 and tgt.tolist() == r["targets"] and loss.tolist() == r["loss_mask"], r["name"]
        _, _, loss2 = oracle.batch_targets(r["tokens"], False)
        assert loss2.tolist() == r["loss_mask_no_tags"], r["name"]
