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


# ---- CacheError::CapacityExceeded on every page-popping path (kvcache.cpp:37-41) ----
# The reference throws before the store changes; the store then stays usable. The engine fast
# paths (append, append_many) must do the same: no host or device state may move on failure.

def _kv_store(mv, pages):
    import torch
    st = mv.kv.PagedStore(num_pages=pages, layers=1, kv_heads=2)
    return st, torch.device("cuda")


def _rand_kv(n, seed):
    import torch
    g = torch.Generator().manual_seed(seed)
    return [((torch.rand(n, 2, 128, generator=g) * 2 - 1).to(torch.bfloat16)).cuda() for _ in range(2)]


def _snapshot(st, hs):
    return [(st.length(h), st.resolve(h), [t.cpu() for t in st.gather_kv(h)]) for h in hs]


def _same(a, b):
    import torch
    assert len(a) == len(b)
    for (la, ta, kva), (lb, tb, kvb) in zip(a, b):
        assert la == lb and ta == tb
        for x, y in zip(kva, kvb):
            assert torch.equal(x, y)


def test_append_exhaustion_raises_and_store_survives(mv):
    import torch
    st, dev = _kv_store(mv, 4)
    h = st.create()
    k, v = _rand_kv(60, 1)
    st.append_many(h, torch.arange(60, dtype=torch.int32, device=dev), torch.arange(60, dtype=torch.int32, device=dev),
                   0, k, v)  # 4 pages, 4 free slots in the tail page
    for t in range(4):
        k1, v1 = _rand_kv(1, 10 + t)
        st.append([h], torch.tensor([100 + t], dtype=torch.int32, device=dev),
                  torch.tensor([60 + t], dtype=torch.int32, device=dev), 0, k1, v1)
    before = _snapshot(st, [h])
    k1, v1 = _rand_kv(1, 99)
    with pytest.raises(mv.CacheError) as e:
        st.append([h], torch.tensor([7], dtype=torch.int32, device=dev), torch.tensor([64], dtype=torch.int32, device=dev),
                  0, k1, v1)
    assert e.value.kind == "CapacityExceeded"
    _same(before, _snapshot(st, [h]))
    assert st.length(h) == 64 and st.resolve(h) == list(range(60)) + [100, 101, 102, 103]
    # a fork shares every page, so its append needs a fresh page too: still refused, nothing moved
    kids = st.fork(h, 2)
    with pytest.raises(mv.CacheError):
        st.append(kids, torch.tensor([8, 9], dtype=torch.int32, device=dev),
                  torch.tensor([64, 64], dtype=torch.int32, device=dev), 0, *_rand_kv(2, 5))
    _same(before * 2, _snapshot(st, kids))
    # releasing the pages makes the same append succeed
    for x in kids + [h]:
        st.release(x)
    s = st.stats()
    assert s.free_pages == 4 and s.total_refcount == 0
    h2 = st.create()
    st.append([h2], torch.tensor([7], dtype=torch.int32, device=dev), torch.tensor([0], dtype=torch.int32, device=dev),
              0, k1, v1)
    assert st.resolve(h2) == [7]
    kk, vv = st.gather_kv(h2)
    assert torch.equal(vv.cpu(), v1.cpu())


def test_append_batch_is_all_or_nothing(mv):
    """A batch where one handle cannot get a page, one is unknown, or one is listed twice changes nothing."""
    import torch
    st, dev = _kv_store(mv, 3)
    a, b = st.create(), st.create()
    st.append_many(a, torch.arange(16, dtype=torch.int32, device=dev), torch.arange(16, dtype=torch.int32, device=dev),
                   0, *_rand_kv(16, 2))  # full page: the next append needs a fresh page
    st.append_many(b, torch.arange(5, dtype=torch.int32, device=dev), torch.arange(5, dtype=torch.int32, device=dev),
                   0, *_rand_kv(5, 3))   # 11 slots left in place
    c = st.fork(a, 1)[0]                 # shares a's full page: needs a fresh page too
    before = _snapshot(st, [a, b, c])
    toks = torch.tensor([50, 51, 52], dtype=torch.int32, device=dev)
    pos = torch.tensor([16, 5, 16], dtype=torch.int32, device=dev)
    with pytest.raises(mv.CacheError) as e:   # two fresh pages wanted, one free
        st.append([a, b, c], toks, pos, 0, *_rand_kv(3, 4))
    assert e.value.kind == "CapacityExceeded"
    _same(before, _snapshot(st, [a, b, c]))
    with pytest.raises(mv.CacheError) as e:   # unknown handle after a valid one
        st.append([b, 987654], toks[:2], pos[:2], 0, *_rand_kv(2, 4))
    assert e.value.kind == "DoubleRelease"
    with pytest.raises(ValueError):          # the same handle twice in one call
        st.append([b, b], toks[:2], pos[:2], 0, *_rand_kv(2, 4))
    _same(before, _snapshot(st, [a, b, c]))
    st.append([a, b], toks[:2], pos[:2], 0, *_rand_kv(2, 4))  # one fresh page: fits
    assert st.resolve(a) == list(range(16)) + [50] and st.resolve(b) == list(range(5)) + [51]
    assert st.resolve(c) == list(range(16))


def test_append_many_exhaustion(mv):
    import torch
    st, dev = _kv_store(mv, 4)
    h = st.create()
    with pytest.raises(mv.CacheError) as e:
        st.append_many(h, torch.arange(65, dtype=torch.int32, device=dev),
                       torch.arange(65, dtype=torch.int32, device=dev), 0, *_rand_kv(65, 6))
    assert e.value.kind == "CapacityExceeded"
    assert st.length(h) == 0 and st.stats().free_pages == 4
    k, v = _rand_kv(64, 7)
    st.append_many(h, torch.arange(64, dtype=torch.int32, device=dev), torch.arange(64, dtype=torch.int32, device=dev),
                   0, k, v)
    assert st.resolve(h) == list(range(64))
    assert torch.equal(st.gather_kv(h)[1].cpu(), v.cpu())


def test_extend_capacity_then_release_recovers(mv):
    """The error is not sticky: after CapacityExceeded a release frees pages and extend succeeds,
    with refcounts conserved (the old device error bit poisoned the store)."""
    st = mv.kv.PagedStore(num_pages=2)
    h = st.extend(st.create(), list(range(32)))
    with pytest.raises(mv.CacheError) as e:
        st.extend(h, [1])
    assert e.value.kind == "CapacityExceeded"
    s = st.stats()
    assert s.total_refcount == 2 and s.free_pages == 0 and s.live_handles == 2
    st.release(h)
    h2 = st.extend(st.create(), list(range(20)))
    assert st.resolve(h2) == list(range(20))
    s = st.stats()
    assert s.total_refcount == 2 and s.free_pages == 0
    with pytest.raises(mv.CacheError):
        st.extend(h2, list(range(13)))  # 12 fit in the tail page, the 13th needs a page
    h3 = st.extend(h2, list(range(12)))
    assert st.length(h3) == 32


def test_merge_precondition_not_fooled_by_lineage(mv):
    """The host proves descent only while the forked prefix is unchanged; other cases go to the
    device slot check (kvcache.cpp:268-274)."""
    st = mv.kv.PagedStore(num_pages=64, record_bytes=0)
    p = st.extend(st.create(), list(range(12)))
    a, b = st.fork(p, 2)
    a2, b2 = st.extend(a, [1, 2]), st.extend(b, [3])
    m = st.merge(p, [a2, b2])                      # proven on the host
    assert st.resolve(m) == list(range(12)) + [1, 2, 3]
    p2 = st.extend(p, [5])                         # a different 13-token prefix
    with pytest.raises(mv.CacheError) as e:
        st.merge(p2, [a2, b2])
    assert e.value.kind == "BranchNotDescendant"
    q = st.extend(st.create(), list(range(12)))    # same tokens, different slots
    with pytest.raises(mv.CacheError) as e:
        st.merge(q, [a2])
    assert e.value.kind == "BranchNotDescendant"
    c = st.extend(p, [9, 9])                       # descends by extend (no fork lineage): device check passes
    m2 = st.merge(p, [c])
    assert st.resolve(m2) == list(range(12)) + [9, 9]
