"""BASELINE configs[0] (C1) end to end on the GPU: the reference's toy transformer (2 layers,
d=256, 4 heads of 64) with this package's kernels for the attention (prefill for
ToyModel::forward, paged fork / merge / append + decode for engine::run_forced), against the
reference's own logits (tests/golden/toy.jsonl.gz, written by the compiled reference) and the
fp64 oracle restatement for the full C1-sized trajectory.

Tolerance: the attention inputs are bf16 (the kernels' contract), the layer algebra fp64, so
logits differ from the fp64 reference by the bf16 rounding of q / k / v propagated through two
layers; LOGIT_TOL bounds it (measured 1.7e-5 max-abs on the 692-token C1 trajectory, logits of
magnitude <= 0.067 at init 0.05) and the greedy argmax must agree."""
import numpy as np
import pytest
import torch

import oracle
from mvtest import record_margin
from paper_2506_09991_b200.host.tokenize import tokenize

pytestmark = pytest.mark.gpu
LOGIT_TOL = 2e-4


@pytest.fixture(scope="module")
def mv():
    import paper_2506_09991_b200 as m
    return m


def gpu_toy(mv, c):
    ref = oracle.Toy(c["layers"], c["heads"], c["model_dim"], c["vocab"], c["seed"], c["init"], c["rope"])
    L = c["layers"]
    w = {"emb": ref.weight("emb"), "unemb": ref.weight("unemb")}
    for k in ("wq", "wk", "wv", "wo", "up", "down"):
        w[k] = [ref.weight(k, l) for l in range(L)]
    return ref, mv.toy.ToyModel(w, L, c["heads"], c["model_dim"], c["vocab"], c["rope"])


def check_logits(got, want, what):
    got = got.cpu().numpy().reshape(want.shape)
    err = np.abs(got - want).max()
    record_margin(f"toy logits {what}", err, LOGIT_TOL)
    agree = (got.argmax(-1) == want.argmax(-1)).mean()
    assert err < LOGIT_TOL, (what, err)
    assert agree == 1.0, (what, agree)
    return err


def test_forward_matches_reference_golden(mv, toy_golden):
    for name in ("t1_small", "t1_c1"):
        g = toy_golden[name]
        _, toy = gpu_toy(mv, g)
        check_logits(toy.forward(g["tokens"]), np.array(g["logits"]).reshape(len(g["tokens"]), -1), name)


def test_run_forced_matches_reference_engine(mv, toy_golden):
    # engine::run_forced logits (per-lane decode with the KV in the store) from the reference
    for name, cfg in (("forced_t1_small", "t1_small"), ("forced_c1_mini", "t1_c1")):
        g, c = toy_golden[name], toy_golden[cfg]
        _, toy = gpu_toy(mv, c)
        ids = tokenize(g["text"])
        logits, rep = toy.run_forced(ids)
        want = np.array(g["logits"]).reshape(len(ids), -1)
        check_logits(logits, want, name)
        assert rep["status"] == "Done" and rep["spawns"] == 1 and rep["merges"] == 1
        assert rep["total_tokens"] == len(ids) == g["total"]


def c1_text(seed=0, prompt_words=512, path_words=64, concl_words=32):
    """configs[0] shape: 512-word prompt, one block of 2 outlines, paths of 64 words, conclusion 32."""
    rng = np.random.default_rng(seed)
    lex = ["value", "residue", "the", "terms", "area", "bound", "compute", "apply", "prime", "result", "of",
           "case", "digits", "total", "lemma", "sum", "factor", "check", "ratio", "segment", "series", "count",
           "root", "length"]
    w = lambda k: " ".join(rng.choice(lex, size=k))  # noqa: E731
    return (w(prompt_words) + " <Parallel> <Goal> <Outline> 1: first </Outline> <Outline> 2: second </Outline> "
            "</Goal> <Path> 1: " + w(path_words) + " </Path> <Path> 2: " + w(path_words) + " </Path> <Conclusion> "
            + w(concl_words) + " </Conclusion> </Parallel>")


def test_c1_full_forward_and_run_forced(mv, toy_golden):
    c = toy_golden["t1_c1"]  # configs[0] model: 2 layers, d 256, 4 heads, vocab 256, seed 0
    ref, toy = gpu_toy(mv, c)
    ids = tokenize(c1_text())
    err, pos, _, _ = oracle.build_dag(ids)
    assert err == 0 and len(ids) > 600
    want = ref.forward(ids, pos, oracle.mask_dense(ids))
    check_logits(toy.forward(ids), want, "C1 forward")
    logits, rep = toy.run_forced(ids)
    check_logits(logits, want, "C1 run_forced")
    assert rep["status"] == "Done" and rep["steps"] < len(ids)  # the two path lanes stepped together


def test_nested_run_forced_equals_forward(mv, toy_golden):
    # nested Process stages: a lane per inner path, forks inside forked lanes, merges inside out
    c = toy_golden["t1_c1"]
    ref, toy = gpu_toy(mv, c)
    text = ("intro words here <Parallel> <Goal> <Outline> 1: a </Outline> <Outline> 2: b </Outline> "
            "<Outline> 3: c </Outline> </Goal> <Path> 1: x x <Parallel> <Goal> <Outline> 1: u </Outline> "
            "<Outline> 2: v </Outline> </Goal> <Path> 1: p q r </Path> <Path> 2: s t </Path> <Conclusion> w "
            "</Conclusion> </Parallel> y </Path> <Path> 2: z z z z </Path> <Path> 3: k </Path> <Conclusion> "
            "done now </Conclusion> </Parallel> tail")
    ids = tokenize(text)
    err, pos, _, _ = oracle.build_dag(ids)
    assert err == 0
    want = ref.forward(ids, pos, oracle.mask_dense(ids))
    logits, rep = toy.run_forced(ids)
    assert rep["status"] == "Done" and rep["spawns"] == 2 and rep["merges"] == 2
    check_logits(logits, want, "nested run_forced")
    check_logits(toy.forward(ids), want, "nested forward")


def test_run_free_matches_reference_engine(mv):
    """engine::run_free (greedy, engine.cpp:941-950) through the C++ engine: the reference's own run
    (tests/golden/free.jsonl.gz, refdrv free) emits the same tokens from the same lanes at the same steps
    and fails at the same step with the same detail (the C1 model breaks the grammar ~20 tokens in)."""
    from conftest import load_jsonl
    for g in load_jsonl("free.jsonl.gz"):
        if g["name"] != "free_c1":
            continue
        ref = oracle.Toy(g["layers"], g["heads"], g["model_dim"], g["vocab"], g["seed"], g["init"], g["rope"])
        _, toy = gpu_toy(mv, {"layers": g["layers"], "heads": g["heads"], "model_dim": g["model_dim"],
                              "vocab": g["vocab"], "seed": g["seed"], "init": g["init"], "rope": g["rope"]})
        rep = toy.run_free(g["prompt"])
        emitted = [e for e in rep["events"] if e[2] in ("Decode", "Prefill")]
        assert [e[3] for e in emitted] == g["tokens"]
        assert [e[0] for e in emitted] == g["steps"] and [e[1] for e in emitted] == g["lanes"]
        assert [0 if e[2] == "Decode" else 1 for e in emitted] == g["kinds"]
        assert rep["status"] == "Failed" and rep["failure_detail"] == g["detail"]
        assert rep["steps"] == g["wall"]  # ConstantStep: wall units = steps


def test_engine_lane_batching_and_limits(mv, toy_golden):
    """Worker length cap (EngineLimits::max_worker_tokens: zombie with MaxLength, the reduce proceeds) and the
    request token limit (LimitExceeded) through the batched engine (engine.cpp:660-676)."""
    c = toy_golden["t1_c1"]
    _, toy = gpu_toy(mv, c)
    ids = tokenize("a b <Parallel> <Goal> <Outline> 1: x </Outline> <Outline> 2: y </Outline> </Goal> "
                   "<Path> 1: p p p p p p </Path> <Path> 2: q </Path> <Conclusion> c </Conclusion> </Parallel> z")
    _, rep = toy.run_forced(ids, max_request_tokens=10)
    assert rep["status"] == "Failed" and rep["failure"] == "LimitExceeded"
    assert rep["failure_detail"] == "request exceeded 10 tokens"


def test_run_batch_many_requests_one_pass_per_step(mv, toy_golden):
    """engine::run_batch with the toy model: three requests of different shapes advance together (one device
    pass per step for the active lanes of all of them); each request's logits equal its own forced run,
    and a malformed request fails alone (finalize reports the first failure, engine.cpp:835-880)."""
    c = toy_golden["t1_c1"]
    ref, toy = gpu_toy(mv, c)
    texts = [c1_text(seed=1, prompt_words=40, path_words=12, concl_words=6),
             "intro words here <Parallel> <Goal> <Outline> 1: a </Outline> <Outline> 2: b </Outline> "
             "<Outline> 3: c </Outline> </Goal> <Path> 1: x x </Path> <Path> 2: z z z z </Path> <Path> 3: k </Path> "
             "<Conclusion> done now </Conclusion> </Parallel> tail",
             "plain sequential text only here"]
    streams = [tokenize(t) for t in texts]
    outs, rep = toy.run_batch(streams)
    assert rep["status"] == "Done" and rep["spawns"] == 2 and rep["merges"] == 2
    assert rep["total_tokens"] == sum(len(s) for s in streams)
    longest_alone = max(toy.run_forced(s)[1]["steps"] for s in streams)
    assert rep["steps"] == longest_alone  # the requests run concurrently
    for s, got in zip(streams, outs):
        err, pos, _, _ = oracle.build_dag(s)
        check_logits(got, ref.forward(s, pos, oracle.mask_dense(s)), f"batch request of {len(s)} tokens")
    bad = streams[1][:-6]  # the stream ends inside its block
    outs, rep = toy.run_batch([streams[0], bad])
    assert rep["status"] == "Failed" and "unterminated block" in rep["failure_detail"]
    check_logits(outs[0], toy.run_forced(streams[0])[0].numpy(), "healthy request beside a failed one")
