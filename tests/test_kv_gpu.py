"""K2 parity: replay the patched reference's RadixStore op logs (tests/golden/kv_*.jsonl.gz)
through the device paged store; every op must return the same handle ids and errors, every
resolve the same tokens and payload bytes (logical-level bit-exactness)."""
import numpy as np
import pytest

from conftest import fnv1a, kv_logs, load_jsonl

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mv():
    import paper_2506_09991_b200 as m
    return m


def payloads_for(prefix, toks, rec):
    """Same rule as oracle/refdrv.cpp payloads_for: FNV-1a of the int32 token prefix."""
    out = bytearray()
    seq = list(prefix)
    for t in toks:
        seq.append(t)
        h = int(fnv1a(np.asarray(seq, np.int32).tobytes()), 16).to_bytes(8, "little")
        out += bytes(h[k % 8] for k in range(rec))
    return bytes(out)


@pytest.mark.parametrize("log", kv_logs())
def test_replay_reference_op_log(mv, log):
    rows = load_jsonl(log)
    rec = rows[0]["record"]
    st = mv.kv.PagedStore(num_pages=4096, record_bytes=rec)
    seqs = {}
    for r in rows[1:-1]:
        op, args = r["op"], r["args"]
        err, res = -1, []
        try:
            if op == "create":
                res = [st.create()]
            elif op == "extend":
                pl = payloads_for(seqs[args[0]], r["tokens"], rec) if rec else None
                res = [st.extend(args[0], r["tokens"], pl)]
            elif op == "fork":
                res = st.fork(args[0], r["n"])
            elif op == "merge":
                res = [st.merge(args[0], args[1:])]
            elif op == "release":
                st.release(args[0])
        except mv.CacheError as e:
            err = {"UnknownHandle": 0, "DoubleRelease": 1, "CapacityExceeded": 2, "BranchNotDescendant": 3}[e.kind]
        assert err == r["error"], (log, r)
        assert res == r["results"], (log, r)
        for rv in r["resolved"]:
            toks = st.resolve(rv["id"])
            assert toks == rv["tokens"], (log, r)
            seqs[rv["id"]] = toks
            assert fnv1a(st.resolve_payloads(rv["id"])) == rv["payload_fnv"], (log, r)
        if op == "release" and err == -1:
            seqs.pop(args[0], None)
    s = st.stats()
    assert s.logical_tokens_reachable == rows[-2]["logical"] and s.live_handles == rows[-2]["live"]
    assert s.bytes_copied_on_last_op == 0
    for rv in rows[-1]["final"]:
        assert st.resolve(rv["id"]) == rv["tokens"]
        assert fnv1a(st.resolve_payloads(rv["id"])) == rv["payload_fnv"]
    # releasing everything returns every page (refcount conservation)
    for rv in rows[-1]["final"]:
        st.release(rv["id"])
    s = st.stats()
    assert s.total_refcount == 0 and s.node_count == 0 and s.free_pages == 4096 and s.live_handles == 0


def test_fork_merge_zero_copy_t1(mv):
    """SPEC.md:252 T1 example: merge(prefix 12, +5, +6) -> length 23, prefix slots shared, 0 bytes."""
    st = mv.kv.PagedStore(num_pages=64, record_bytes=8)
    root = st.create()
    p = st.extend(root, list(range(10, 22)), bytes(96))
    a, b = st.fork(p, 2)
    free_before = st.stats().free_pages
    a2 = st.extend(a, [30, 31, 32, 33, 34], bytes(40))
    b2 = st.extend(b, [40, 41, 42, 43, 44, 45], bytes(48))
    pages_for_branches = free_before - st.stats().free_pages
    m = st.merge(p, [a2, b2])
    assert st.length(m) == 23
    assert st.resolve(m) == list(range(10, 22)) + [30, 31, 32, 33, 34] + [40, 41, 42, 43, 44, 45]
    sp, sa, sb, sm = (st.resolve_slots(h) for h in (p, a2, b2, m))
    assert sm == sp + sa[12:] + sb[12:]  # index concatenation: every merged slot is an existing slot
    assert st.stats().free_pages == 64 - 1 - pages_for_branches  # merge allocated no page
    assert st.stats().bytes_copied_on_last_op == 0
    with pytest.raises(mv.CacheError) as e:
        st.merge(a2, [p])
    assert e.value.kind == "BranchNotDescendant"
    with pytest.raises(mv.CacheError) as e:
        st.release(12345)
    assert e.value.kind == "DoubleRelease"


def test_capacity_exceeded(mv):
    st = mv.kv.PagedStore(num_pages=2, record_bytes=0)
    h = st.create()
    h2 = st.extend(h, list(range(32)))
    assert st.length(h2) == 32
    with pytest.raises(mv.CacheError) as e:
        st.extend(h2, [1])
    assert e.value.kind == "CapacityExceeded"


def test_refcount_conservation_fork_release(mv):
    st = mv.kv.PagedStore(num_pages=128)
    h = st.extend(st.create(), list(range(100)))  # 7 pages -> 7 entries
    base = st.stats().total_refcount
    kids = st.fork(h, 5)
    assert st.stats().total_refcount == base + 5 * 7  # +n per shared entry (SPEC.md kvcache invariants)
    assert st.stats().physical_tokens_stored == 100   # fork stores nothing new
    for k in kids:
        st.release(k)
    assert st.stats().total_refcount == base
