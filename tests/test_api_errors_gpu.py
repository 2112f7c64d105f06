"""Error behaviour of the attention and store entry points (the reference throws
std::invalid_argument for shape errors, toy_model.cpp:47-51 / :90-92 / :177-179, and
CacheError{DoubleRelease} for unknown handles, kvcache.cpp:16-20): every bad call raises the
mirrored exception and leaves the store usable."""
import pytest
import torch

from mvtest import sym_bf16

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mv():
    import paper_2506_09991_b200 as m
    return m


@pytest.fixture()
def store(mv):
    st = mv.kv.PagedStore(num_pages=64, layers=2, kv_heads=2)
    h = st.create()
    k, v = sym_bf16(1, (20, 2, 128)).cuda(), sym_bf16(2, (20, 2, 128)).cuda()
    st.append_many(h, torch.full((20,), 11, dtype=torch.int32, device="cuda"),
                   torch.arange(20, dtype=torch.int32, device="cuda"), 0, k, v)
    return st, h


def test_decode_rejects_bad_shapes_and_handles(mv, store):
    st, h = store
    q = sym_bf16(3, (1, 4, 128)).cuda()
    pos = torch.tensor([19], dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):  # q_heads not a multiple of kv_heads
        mv.attention.decode(st, [h], sym_bf16(4, (1, 3, 128)).cuda(), pos)
    with pytest.raises(ValueError):  # no attention plane for layer 5
        mv.attention.decode(st, [h], q, pos, layer=5)
    with pytest.raises(mv.CacheError) as e:  # unknown handle -> DoubleRelease, as the reference
        mv.attention.decode(st, [h + 999], q, pos)
    assert e.value.kind == "DoubleRelease"
    empty = st.create()
    with pytest.raises(ValueError):  # nothing to attend to
        mv.attention.decode(st, [empty], q, pos)
    out = mv.attention.decode(st, [h], q, pos)  # the store still works
    torch.cuda.synchronize()
    assert bool(torch.isfinite(out.float()).all())


def test_release_twice_and_merge_non_descendant(mv, store):
    st, h = store
    kids = st.fork(h, 2)
    other = st.create()
    st.append_many(other, torch.full((3,), 12, dtype=torch.int32, device="cuda"), None, 0, None, None, n=3)
    with pytest.raises(mv.CacheError) as e:
        st.merge(h, [kids[0], other])
    assert e.value.kind == "BranchNotDescendant"
    st.release(kids[1])
    with pytest.raises(mv.CacheError) as e:
        st.release(kids[1])
    assert e.value.kind == "DoubleRelease"
    m = st.merge(h, [kids[0]])
    assert st.length(m) == st.length(h)


def test_prefill_rejects_bad_arguments(mv):
    toks = [11, 12, 13, 14]
    spec = mv.dag.build_visibility(toks)
    q, k, v = sym_bf16(5, (4, 4, 128)).cuda(), sym_bf16(6, (4, 2, 128)).cuda(), sym_bf16(7, (4, 2, 128)).cuda()
    with pytest.raises(ValueError):  # q heads not a multiple of kv heads
        mv.attention.prefill(sym_bf16(8, (4, 3, 128)).cuda(), k, v, spec.positions, spec.excl)
    out = mv.attention.prefill(q, k, v, spec.positions, spec.excl)
    torch.cuda.synchronize()
    assert bool(torch.isfinite(out.float()).all())


def test_handle_arrays_match_lists(mv):
    """kv.handle_array (zero-copy uint64 handles) and plain lists give identical results."""
    import numpy as np
    outs = []
    for as_array in (False, True):
        st = mv.kv.PagedStore(num_pages=128, layers=1, kv_heads=2)
        root = st.create()
        k, v = sym_bf16(11, (40, 2, 128)).cuda(), sym_bf16(12, (40, 2, 128)).cuda()
        st.append_many(root, torch.full((40,), 11, dtype=torch.int32, device="cuda"),
                       torch.arange(40, dtype=torch.int32, device="cuda"), 0, k, v)
        kids = st.fork(root, 3)
        hs = mv.kv.handle_array(kids) if as_array else list(kids)
        pos = torch.full((3,), 40, dtype=torch.int32, device="cuda")
        st.append(hs, torch.full((3,), 12, dtype=torch.int32, device="cuda"), pos, 0,
                  sym_bf16(13, (3, 2, 128)).cuda(), sym_bf16(14, (3, 2, 128)).cuda())
        outs.append(mv.attention.decode(st, hs, sym_bf16(15, (3, 4, 128)).cuda(), pos, out_dtype=torch.float32))
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    assert isinstance(mv.kv.handle_array([1, 2]), np.ndarray)
