"""K5 — per-lane tag interpreter (engine.cpp:323-415 feed_interpreter, BUG-2 fixed; merge reset
engine.cpp:793).

CPU: the Python restatement (oracle/interp.py) reproduces the reference's own interpreter on
every stream of tests/golden/interp.jsonl.gz (actions, spawn counts, frame state after each
event, violation texts). GPU: the device kernel, all golden streams as lanes of one launch and
again one event per launch, reproduces the same actions / arguments / violation texts / final
state bit-exactly, plus a 16K-lane random run against the restatement."""
import numpy as np
import pytest
import torch

from conftest import load_jsonl
from oracle import interp as ointerp


@pytest.fixture(scope="module")
def golden():
    return load_jsonl("interp.jsonl.gz")


def test_oracle_matches_reference_interpreter(golden):
    assert len(golden) > 1500
    for g in golden:
        rows, det = ointerp.run(g["child"], g["events"])
        assert rows == g["out"], g["events"]
        assert det == {int(k): v for k, v in g["detail"].items()}, g["events"]
    kinds = {r[0] for g in golden for r in g["out"]}
    assert kinds == {0, 1, 2, 3}


def lanes_matrix(golden):
    n = len(golden)
    steps = max(len(g["events"]) for g in golden)
    ev = np.full((steps, n), -1, np.int32)  # IDLE past a stream's end
    for j, g in enumerate(golden):
        ev[: len(g["events"]), j] = g["events"]
    return ev, np.array([g["child"] for g in golden], np.int32)


def check_against_golden(mv, golden, action, arg, it):
    action, arg = action.cpu().numpy(), arg.cpu().numpy()
    for j, g in enumerate(golden):
        n = len(g["events"])
        out = np.array(g["out"], np.int64).reshape(n, 7)
        bad = np.nonzero(action[:n, j] != out[:, 0])[0]
        assert bad.size == 0, (j, g["child"], g["events"], bad[:3].tolist(), action[:n, j].tolist(), out[:, 0].tolist())
        spawn = out[:, 0] == mv.interp.SPAWN
        assert (arg[:n, j][spawn] == out[spawn, 1]).all()
        assert (action[n:, j] == mv.interp.NONE).all()  # idle steps
        texts = {i: mv.interp.violation_text(int(arg[i, j]), g["events"][i])
                 for i in range(n) if action[i, j] == mv.interp.VIOLATION}
        assert texts == {int(k): v for k, v in g["detail"].items()}, j
    final = it.lanes().cpu().numpy()
    want = np.array([g["out"][-1][2:] for g in golden])
    assert (final == want).all()


@pytest.mark.gpu
def test_device_one_launch_matches_reference(golden):
    import paper_2506_09991_b200 as mv
    ev, child = lanes_matrix(golden)
    it = mv.interp.TagInterpreter(len(golden), child)
    action, arg, sp, cnt = it.feed(torch.from_numpy(ev), spawns=True)
    check_against_golden(mv, golden, action, arg, it)
    # compacted spawn list == the spawn events, as a set
    k = int(cnt.item())
    got = sorted(map(tuple, sp[:k].cpu().numpy().tolist()))
    want = sorted((i, j, r[1]) for j, g in enumerate(golden) for i, r in enumerate(g["out"]) if r[0] == 1)
    assert got == want


@pytest.mark.gpu
def test_device_step_by_step_matches_reference(golden):
    import paper_2506_09991_b200 as mv
    ev, child = lanes_matrix(golden)
    it = mv.interp.TagInterpreter(len(golden), child)
    d = torch.from_numpy(ev).cuda()
    acts, args = zip(*(it.feed(d[s]) for s in range(d.shape[0])))  # one launch per decode step
    check_against_golden(mv, golden, torch.stack(acts), torch.stack(args), it)


@pytest.mark.gpu
def test_device_random_lanes_against_restatement():
    import paper_2506_09991_b200 as mv
    rng = np.random.default_rng(11)
    n, steps = 16384, 48
    pool = np.array([*range(10), 10, 11, 12, 13, -1, -2], np.int32)
    w = np.array([3, 1, 3, 2, 4, 4, 2, 2, 2, 2, 3, 3, 3, 3, 2, 1], np.float64)
    ev = rng.choice(pool, size=(steps, n), p=w / w.sum()).astype(np.int32)
    child = rng.integers(0, 2, n).astype(np.int32)
    it = mv.interp.TagInterpreter(n, child)
    a1, r1 = it.feed(torch.from_numpy(ev[:20]))
    a2, r2 = it.feed(torch.from_numpy(ev[20:]))  # state carried across launches
    action = torch.cat([a1, a2]).cpu().numpy()
    arg = torch.cat([r1, r2]).cpu().numpy()
    final = it.lanes().cpu().numpy()
    for j in range(0, n, 7):  # a seventh of the lanes through the pure-Python restatement
        rows, det = ointerp.run(child[j], ev[:, j])
        rows = np.array(rows)
        bad = np.nonzero(action[:, j] != rows[:, 0])[0]
        assert bad.size == 0, (j, int(child[j]), ev[:, j].tolist(), bad[:3].tolist(), action[:, j].tolist(),
                               rows[:, 0].tolist())
        sp = rows[:, 0] == 1
        assert (arg[sp, j] == rows[sp, 1]).all()
        assert {i: mv.interp.violation_text(int(arg[i, j]), int(ev[i, j])) for i in det} == det
        assert (final[j] == rows[-1, 2:]).all()


@pytest.mark.gpu
def test_device_argument_errors():
    import paper_2506_09991_b200 as mv
    with pytest.raises(ValueError):
        mv.interp.TagInterpreter(4, [0, 1])
    it = mv.interp.TagInterpreter(0)
    a, r = it.feed(torch.zeros((3, 0), dtype=torch.int32))
    assert a.numel() == 0
