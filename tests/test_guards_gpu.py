"""Out-of-bounds write checks of our own (compute-sanitizer is closed on this GPU pool: runs under it left
GPUs needing a reset).  Every output is a view into a larger buffer filled with a sentinel bit pattern; the
kernels must write exactly the view and leave every guard element bit-identical, and the page pool must keep
the K/V of a bystander handle that no call touches.  Cases cover the decode unit kinds (plain, row-copied,
split-KV with partial slots, single-context combine), the fp32 and bf16 stores, masked prefill with ragged
tiles, and the page-popping append paths next to a bystander."""
import numpy as np
import pytest
import torch

from mvtest import sym_bf16

pytestmark = pytest.mark.gpu
GUARD = 4096  # elements on each side of the view


@pytest.fixture(scope="module")
def mv():
    import paper_2506_09991_b200 as m
    return m


def guarded(shape, dtype):
    n = int(np.prod(shape))
    buf = torch.empty(n + 2 * GUARD, dtype=dtype, device="cuda")
    buf.view(torch.int16 if dtype == torch.bfloat16 else torch.int32).fill_(0x7F7B if dtype == torch.bfloat16 else 0x7F7BCDEF)
    return buf, buf[GUARD:GUARD + n].view(*shape)


def guards_intact(buf, dtype):
    iv = buf.view(torch.int16 if dtype == torch.bfloat16 else torch.int32)
    pat = 0x7F7B if dtype == torch.bfloat16 else 0x7F7BCDEF
    return bool((iv[:GUARD] == pat).all()) and bool((iv[-GUARD:] == pat).all())


def build(mv, specs, hkv=8, num_pages=4096, seed=5):
    """specs: (prefix, branches, branch_len) per request -> store, handles, next positions, bystander."""
    dev = "cuda"
    st = mv.kv.PagedStore(num_pages=num_pages, layers=1, kv_heads=hkv)
    hs, pos = [], []
    for i, (prefix, branches, blen) in enumerate(specs):
        root = st.create()
        k, v = sym_bf16(seed + 10 * i, (prefix, hkv, 128)), sym_bf16(seed + 10 * i + 1, (prefix, hkv, 128))
        st.append_many(root, torch.full((prefix,), 11, dtype=torch.int32, device=dev),
                       torch.arange(prefix, dtype=torch.int32, device=dev), 0, k.to(dev), v.to(dev))
        for j, h in enumerate(st.fork(root, branches)):
            kb, vb = sym_bf16(seed + 100 * i + j, (blen, hkv, 128)), sym_bf16(seed + 100 * i + j + 50, (blen, hkv, 128))
            st.append_many(h, torch.full((blen,), 12, dtype=torch.int32, device=dev),
                           torch.arange(prefix, prefix + blen, dtype=torch.int32, device=dev), 0, kb.to(dev), vb.to(dev))
            hs.append(h)
            pos.append(prefix + blen)
    by = st.create()  # a bystander with a partially filled tail page
    kb, vb = sym_bf16(seed + 999, (37, hkv, 128)), sym_bf16(seed + 998, (37, hkv, 128))
    st.append_many(by, torch.full((37,), 13, dtype=torch.int32, device=dev), torch.arange(37, dtype=torch.int32, device=dev),
                   0, kb.to(dev), vb.to(dev))
    return st, hs, pos, by


@pytest.mark.parametrize("specs,hq,hkv", [
    ([(200, 3, 40)], 40, 8),                       # small plain units
    ([(1000, 8, 300), (64, 2, 17)], 40, 8),        # F = 2 row copies (8 x 5 rows), ragged pages
    ([(4096, 32, 100)], 40, 8),                    # > 16 members: split member groups
    ([(16, 1, 9000)], 40, 8),                      # one long context: split-KV slots + combine
    ([(333, 4, 70)], 8, 8),                        # MHA
])
@pytest.mark.parametrize("odt", [torch.float32, torch.bfloat16])
def test_decode_writes_only_its_output(mv, specs, hq, hkv, odt):
    st, hs, pos, by = build(mv, specs, hkv=hkv)
    n = len(hs)
    before = [x.clone() for x in st.gather_kv(by)]
    p = torch.tensor(pos, dtype=torch.int32, device="cuda")
    st.append(hs, torch.full((n,), 12, dtype=torch.int32, device="cuda"), p, 0,
              sym_bf16(7, (n, hkv, 128)).cuda(), sym_bf16(8, (n, hkv, 128)).cuda())
    q = sym_bf16(9, (n, hq, 128)).cuda()
    buf, out = guarded((n, hq, 128), odt)
    mv.attention.decode(st, hs, q, p, out=out)
    torch.cuda.synchronize()
    assert guards_intact(buf, odt)
    assert bool(torch.isfinite(out.float()).all())
    after = st.gather_kv(by)
    assert all(torch.equal(a, b) for a, b in zip(before, after))


@pytest.mark.parametrize("n", [1, 127, 129, 1000])
@pytest.mark.parametrize("odt", [torch.float32, torch.bfloat16])
def test_prefill_writes_only_its_output(mv, n, odt):
    from test_prefill_gpu import nested_tokens
    toks = nested_tokens(2, 3, 40, seed=n) if n > 200 else list(range(30, 30 + n))
    n = len(toks)
    spec = mv.dag.build_visibility(toks)
    q, k, v = sym_bf16(1, (n, 40, 128)).cuda(), sym_bf16(2, (n, 8, 128)).cuda(), sym_bf16(3, (n, 8, 128)).cuda()
    ref = mv.attention.prefill(q, k, v, spec.positions, spec.excl, out_dtype=odt)
    buf, out = guarded((n, 40, 128), odt)
    mv.attention.prefill(q, k, v, spec.positions, spec.excl, out=out)
    torch.cuda.synchronize()
    assert guards_intact(buf, odt)
    assert torch.equal(out, ref)


def test_append_paths_leave_bystander_pages(mv):
    """append / append_many / extend popping fresh pages (and failing with CapacityExceeded at the end) never
    write a page another handle holds."""
    st, hs, pos, by = build(mv, [(40, 3, 16)], num_pages=40)
    before = [x.clone() for x in st.gather_kv(by)]
    dev = "cuda"
    p = torch.tensor(pos, dtype=torch.int32, device=dev)
    for step in range(200):
        try:
            st.append(hs, torch.full((3,), 12, dtype=torch.int32, device=dev), p + step, 0,
                      sym_bf16(step, (3, 8, 128)).cuda(), sym_bf16(step + 1, (3, 8, 128)).cuda())
        except mv.CacheError as e:
            assert e.kind == "CapacityExceeded"
            break
    else:
        pytest.fail("pool never ran out")
    with pytest.raises(mv.CacheError):
        st.append_many(hs[0], torch.full((64,), 5, dtype=torch.int32, device=dev),
                       torch.arange(64, dtype=torch.int32, device=dev), 0, sym_bf16(3, (64, 8, 128)).cuda(),
                       sym_bf16(4, (64, 8, 128)).cuda())
    torch.cuda.synchronize()
    after = st.gather_kv(by)
    assert all(torch.equal(a, b) for a, b in zip(before, after))
    assert st.resolve(by) == [13] * 37
