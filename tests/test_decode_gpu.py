"""K4 parity: branch-parallel paged decode attention vs the fp64 oracle restatement of
toy_model.cpp:121-157 (GQA h -> h/(Hq/Hkv)), on bf16-rounded seeded inputs.
Tolerance (north star): max-abs 2e-3 with fp32 accumulation."""
import numpy as np
import pytest
import torch

import oracle
from mvtest import bf16_to_f64, record_margin, sym_bf16

pytestmark = pytest.mark.gpu
TOL = 2e-3


@pytest.fixture(scope="module")
def mv():
    import paper_2506_09991_b200 as m
    return m


class Req:
    """One request: shared prefix, fork into branches, per-branch private tokens, one decode step."""

    def __init__(self, mv, st, rows, seed, prefix, branches, branch_len, hkv, nested=None, spike=False, d=128):
        self.st, self.rows = st, rows
        dev = "cuda"

        def add(h, n, pos0, private=False):
            k = sym_bf16(seed * 1000 + len(rows["k"]) * 7 + 1, (n, hkv, d))
            if spike and private:
                # the middle key of a branch's private run scores ~260 log2 units above the rest of the
                # branch's context (dims 124-127 barely rotate: theta ~1e-4 rad per position)
                k[n // 2, :, :] = 0.0
                k[n // 2, :, d - 4:] = 512.0
            v = sym_bf16(seed * 1000 + len(rows["k"]) * 7 + 2, (n, hkv, d))
            pos = torch.arange(pos0, pos0 + n, dtype=torch.int32)
            st.append_many(h, torch.full((n,), 11, dtype=torch.int32, device=dev), pos.to(dev), 0, k.to(dev),
                           v.to(dev))
            base = sum(x.shape[0] for x in rows["k"])
            rows["k"].append(k)
            rows["v"].append(v)
            rows["pos"].append(pos)
            return list(range(base, base + n))

        root = st.create()
        ctx_root = add(root, prefix, 0) if prefix else []
        self.handles, self.ctx, self.qpos = [], [], []
        kids = st.fork(root, branches)
        for i, h in enumerate(kids):
            if nested and i == 0:
                # nested Process stage inside branch 0: extend, fork again
                c = ctx_root + add(h, nested[0], prefix)
                sub = st.fork(h, nested[1])
                for s in sub:
                    cc = c + add(s, branch_len - 1, prefix + nested[0])
                    self.handles.append(s)
                    self.ctx.append(cc)
                    self.qpos.append(prefix + nested[0] + branch_len - 1)
                continue
            c = ctx_root + (add(h, branch_len - 1, prefix, private=True) if branch_len > 1 else [])
            self.handles.append(h)
            self.ctx.append(c)
            self.qpos.append(prefix + branch_len - 1)
        self.root, self.ctx_root = root, ctx_root


def run_case(mv, reqs_spec, hq, hkv, num_pages, seed=1, spike=False, d=128):
    st = mv.kv.PagedStore(num_pages=num_pages, layers=1, kv_heads=hkv, head_dim=d)
    rows = {"k": [], "v": [], "pos": []}
    reqs = [Req(mv, st, rows, seed + i, *spec, hkv=hkv, spike=spike, d=d) if len(spec) == 3 else
            Req(mv, st, rows, seed + i, *spec[:3], hkv=hkv, nested=spec[3], d=d) for i, spec in enumerate(reqs_spec)]
    handles = [h for r in reqs for h in r.handles]
    ctx = [c for r in reqs for c in r.ctx]
    qpos = [p for r in reqs for p in r.qpos]
    n = len(handles)
    # the decode step: append each branch's new token (K/V), then attend
    knew = sym_bf16(seed * 77 + 5, (n, hkv, d))
    vnew = sym_bf16(seed * 77 + 6, (n, hkv, d))
    q = sym_bf16(seed * 77 + 7, (n, hq, d))
    if spike:
        q[:, :, d - 4:] = 1.0
    pos = torch.tensor(qpos, dtype=torch.int32)
    st.append(handles, torch.full((n,), 12, dtype=torch.int32, device="cuda"), pos.cuda(), 0, knew.cuda(),
              vnew.cuda())
    out = mv.attention.decode(st, handles, q.cuda(), pos.cuda(), out_dtype=torch.float32)
    torch.cuda.synchronize()
    # oracle: rotate K at cache time and q at its position (fp64), attend prefix..suffix..self
    base = sum(x.shape[0] for x in rows["k"])
    K = np.concatenate([bf16_to_f64(x) for x in rows["k"]] + [bf16_to_f64(knew)])
    V = np.concatenate([bf16_to_f64(x) for x in rows["v"]] + [bf16_to_f64(vnew)])
    P = np.concatenate([x.numpy() for x in rows["pos"]] + [pos.numpy()])
    Kr = oracle.rope(K, P)
    qr = oracle.rope(bf16_to_f64(q), pos.numpy())
    ctx_full = [c + [base + i] for i, c in enumerate(ctx)]
    ref = oracle.attn_decode(qr, Kr, V, ctx_full)
    err = np.abs(out.float().cpu().numpy() - ref).max()
    record_margin(f"decode {len(handles)} handles hq={hq}/{hkv}" + (f" d={d}" if d != 128 else ""), err, TOL)
    # the bf16 output path: identical arithmetic plus the bf16 store rounding (<= 2^-9 |o|)
    out16 = mv.attention.decode(st, handles, q.cuda(), pos.cuda()).float().cpu().numpy()
    assert (np.abs(out16 - ref) <= TOL + np.abs(ref) * 2.0 ** -8).all()
    return err, st


def test_small_gqa(mv):
    err, st = run_case(mv, [(300, 3, 37)], hq=8, hkv=2, num_pages=256)
    assert err < TOL, err
    info = st.plan_info()
    assert info["unique_kv_tokens"] < info["naive_kv_tokens"]  # the prefix is read once


def test_score_spike(mv):
    """One key in the middle of every branch's private run dwarfs the rest of its context: the softmax
    reference must move (sum guard) even on polynomial-exp2 columns; branch lengths 600..615 walk the key
    across the columns of its block."""
    err, _ = run_case(mv, [(700, 2, 600 + i) for i in range(16)], hq=8, hkv=1, num_pages=2048, spike=True)
    assert err < TOL, err


@pytest.mark.parametrize("blen", [1, 17, 33, 49, 65, 130, 257])
def test_narrow_units(mv, blen):
    """Private tails of 1..17 blocks (<= 32 query rows in one lane quadrant), including units shorter than the
    S ring; the single-context case (no prefix) is written by the epilogue directly, the forked ones through
    the split-KV combine."""
    err, _ = run_case(mv, [(0, 1, blen), (64, 3, blen), (500, 2, blen + 3)], hq=40, hkv=8, num_pages=512,
                      seed=blen)
    assert err < TOL, err
    err, _ = run_case(mv, [(40, 2, blen)], hq=16, hkv=1, num_pages=256, seed=blen + 1)  # R = 16 rows per member
    assert err < TOL, err


def test_ragged_unaligned_prefix(mv):
    # prefix length not a multiple of 16: the shared tail page is partial
    err, _ = run_case(mv, [(77, 4, 19), (5, 2, 3), (0, 2, 1)], hq=40, hkv=8, num_pages=256)
    assert err < TOL, err


def test_nested_fork_lineage(mv):
    # branch 0 forks again: a 2-level cascade (prefix shared by all, mid segment by 3)
    err, st = run_case(mv, [(200, 3, 30, (40, 3))], hq=40, hkv=8, num_pages=512)
    assert err < TOL, err


def test_many_members_row_split(mv):
    # 20 branches x 5 heads = 100 rows per KV head: split across CTAs (L2 re-reads)
    err, _ = run_case(mv, [(130, 20, 9)], hq=40, hkv=8, num_pages=512)
    assert err < TOL, err


def test_c2_shape(mv):
    # BASELINE configs[1]: 40 q / 8 kv heads, 4K shared prefix, 8 branches x 1K, page 16
    err, st = run_case(mv, [(4096, 8, 1024)], hq=40, hkv=8, num_pages=1024)
    assert err < TOL, err
    info = st.plan_info()
    assert info["unique_kv_tokens"] == 4096 + 8 * 1024
    assert info["naive_kv_tokens"] == 8 * (4096 + 1024)


def test_decode_after_merge(mv):
    """Reduce stage: zero-copy merge of the branches, then keep decoding over the merged KV
    (engine.cpp:767-802 then emit over the merged handle)."""
    hq, hkv = 40, 8
    st = mv.kv.PagedStore(num_pages=256, layers=1, kv_heads=hkv)
    rows = {"k": [], "v": [], "pos": []}
    r = Req(mv, st, rows, 9, 100, 3, 20, hkv=hkv)
    m = st.merge(r.root, r.handles)
    ctx = list(r.ctx_root)
    for c in r.ctx:
        ctx += c[len(r.ctx_root):]
    assert st.length(m) == len(ctx)
    for h in r.handles + [r.root]:
        st.release(h)  # zombies released after the merge; pages stay alive through m
    knew, vnew, q = sym_bf16(555, (1, hkv, 128)), sym_bf16(556, (1, hkv, 128)), sym_bf16(557, (1, hq, 128))
    pos = torch.tensor([100 + 19], dtype=torch.int32)  # max path end + 1
    st.append([m], torch.tensor([13], dtype=torch.int32, device="cuda"), pos.cuda(), 0, knew.cuda(), vnew.cuda())
    out = mv.attention.decode(st, [m], q.cuda(), pos.cuda(), out_dtype=torch.float32)
    base = sum(x.shape[0] for x in rows["k"])
    K = np.concatenate([bf16_to_f64(x) for x in rows["k"]] + [bf16_to_f64(knew)])
    V = np.concatenate([bf16_to_f64(x) for x in rows["v"]] + [bf16_to_f64(vnew)])
    P = np.concatenate([x.numpy() for x in rows["pos"]] + [pos.numpy()])
    ref = oracle.attn_decode(oracle.rope(bf16_to_f64(q), pos.numpy()), oracle.rope(K, P), V, [ctx + [base]])
    assert np.abs(out.float().cpu().numpy() - ref).max() < TOL


def test_many_requests_persistent_mix(mv):
    # > 148 (item, kv head) work units: every persistent CTA runs several mixed-width items
    # back to back (cascade prefix items + private items), exercising the ring hand-over.
    err, st = run_case(mv, [(1024, 8, 200)] * 8 + [(333, 3, 77)] * 3, hq=40, hkv=8, num_pages=2048, seed=5)
    assert err < TOL, err
    assert st.plan_info()["work_items"] * 8 > 148


def test_multi_step_decode_growing_tables(mv):
    """Engine loop: 40 decode steps per branch (append then attend), crossing page boundaries, so
    the cached decode plan is updated in place (tail chunks grow) and re-planned when a chunk fills;
    every step is checked against the oracle."""
    hq, hkv = 40, 8
    st = mv.kv.PagedStore(num_pages=512, layers=1, kv_heads=hkv)
    rows = {"k": [], "v": [], "pos": []}
    r = Req(mv, st, rows, 11, 1000, 4, 1013, hkv=hkv)  # tails end 3 tokens before a page boundary
    handles, ctx, qpos = list(r.handles), [list(c) for c in r.ctx], list(r.qpos)
    n = len(handles)
    for step in range(40):
        knew = sym_bf16(9000 + step * 3, (n, hkv, 128))
        vnew = sym_bf16(9001 + step * 3, (n, hkv, 128))
        q = sym_bf16(9002 + step * 3, (n, hq, 128))
        pos = torch.tensor(qpos, dtype=torch.int32)
        st.append(handles, torch.full((n,), 12, dtype=torch.int32, device="cuda"), pos.cuda(), 0, knew.cuda(),
                  vnew.cuda())
        base = sum(x.shape[0] for x in rows["k"])
        rows["k"].append(knew)
        rows["v"].append(vnew)
        rows["pos"].append(pos)
        for i in range(n):
            ctx[i].append(base + i)
        out = mv.attention.decode(st, handles, q.cuda(), pos.cuda(), out_dtype=torch.float32)
        if step % 7 == 0 or step == 39:
            K = np.concatenate([bf16_to_f64(x) for x in rows["k"]])
            V = np.concatenate([bf16_to_f64(x) for x in rows["v"]])
            P = np.concatenate([x.numpy() for x in rows["pos"]])
            ref = oracle.attn_decode(oracle.rope(bf16_to_f64(q), pos.numpy()), oracle.rope(K, P), V, ctx)
            err = np.abs(out.float().cpu().numpy() - ref).max()
            assert err < TOL, (step, err)
        qpos = [p + 1 for p in qpos]


def test_reduce_merge_stress_then_decode(mv):
    """BASELINE configs[4] in miniature: R rounds of {fork B branches; each branch appends a path;
    zero-copy merge in ordinal order; append the Reduce tokens}, then decode over the merged KV
    (engine.cpp:679-725 spawn, :767-802 merge).  Checks 0 bytes copied and no page allocated by
    fork / merge, refcount conservation, and decode parity against the oracle."""
    hq, hkv, B, R, path, red = 40, 8, 24, 4, 17, 5
    st = mv.kv.PagedStore(num_pages=2048, layers=1, kv_heads=hkv)
    rows = {"k": [], "v": [], "pos": []}
    seed = [100]

    def add(h, n, pos0):
        seed[0] += 2
        k = sym_bf16(seed[0], (n, hkv, 128))
        v = sym_bf16(seed[0] + 1, (n, hkv, 128))
        pos = torch.arange(pos0, pos0 + n, dtype=torch.int32)
        st.append_many(h, torch.full((n,), 11, dtype=torch.int32, device="cuda"), pos.cuda(), 0, k.cuda(), v.cuda())
        base = sum(x.shape[0] for x in rows["k"])
        rows["k"].append(k)
        rows["v"].append(v)
        rows["pos"].append(pos)
        return list(range(base, base + n))

    cur = st.create()
    ctx = add(cur, 250, 0)
    L = 250
    for _ in range(R):
        kids = st.fork(cur, B)
        s0 = st.stats()
        assert s0.bytes_copied_on_last_op == 0
        kid_ctx = [add(k, path, L) for k in kids]  # sibling paths share their start position
        free_before = st.stats().free_pages
        m = st.merge(cur, kids)
        s1 = st.stats()
        assert s1.bytes_copied_on_last_op == 0 and s1.free_pages == free_before  # merge moves no KV, allocates no page
        ctx = ctx + [r for kc in kid_ctx for r in kc]
        for h in [cur] + kids:
            st.release(h)
        L += path  # Reduce starts at max path end + 1
        ctx = ctx + add(m, red, L)
        L += red
        cur = m
        assert st.length(cur) == len(ctx)
    assert st.resolve_slots(cur) is not None
    for step in range(3):
        knew, vnew, q = sym_bf16(7000 + step, (1, hkv, 128)), sym_bf16(7100 + step, (1, hkv, 128)), sym_bf16(7200 + step, (1, hq, 128))
        pos = torch.tensor([L], dtype=torch.int32)
        st.append([cur], torch.tensor([13], dtype=torch.int32, device="cuda"), pos.cuda(), 0, knew.cuda(), vnew.cuda())
        base = sum(x.shape[0] for x in rows["k"])
        rows["k"].append(knew)
        rows["v"].append(vnew)
        rows["pos"].append(pos)
        ctx = ctx + [base]
        out = mv.attention.decode(st, [cur], q.cuda(), pos.cuda(), out_dtype=torch.float32)
        K = np.concatenate([bf16_to_f64(x) for x in rows["k"]])
        V = np.concatenate([bf16_to_f64(x) for x in rows["v"]])
        P = np.concatenate([x.numpy() for x in rows["pos"]])
        ref = oracle.attn_decode(oracle.rope(bf16_to_f64(q), pos.numpy()), oracle.rope(K, P), V, [ctx])
        assert np.abs(out.float().cpu().numpy() - ref).max() < TOL
        L += 1
    st.release(cur)
    s = st.stats()
    assert s.live_handles == 0 and s.total_refcount == 0 and s.free_pages == 2048


def test_c4_full_scale_sampled(mv):
    """BASELINE configs[3] at full size on one GPU: 64 requests x 32 branches, 16K shared prefix +
    32 x 512 branch tokens (32K unique per request, 8.6 GB of bf16 K/V), one decode step for all
    2,048 branches.  Size-independent checks on the whole batch (plan reads every unique token
    once per member group, finite outputs), oracle parity on a seeded sample of branches."""
    hq, hkv, R, B, prefix, blen = 40, 8, 64, 32, 16384, 512
    pages = R * (prefix // 16 + 1 + B * (blen // 16 + 3)) + 1024
    table = 2 * R * (B + 1) * (prefix // 16 + blen // 16 + 8) + 65536
    st = mv.kv.PagedStore(num_pages=pages, layers=1, kv_heads=hkv, table_entries=table)
    sample = {3: [0, 17, 31], 50: [5, 30]}  # request -> branches checked against the oracle
    kept = {}
    handles, qpos = [], []
    for r in range(R):
        g = torch.Generator(device="cuda")
        g.manual_seed(4242 + r)
        rnd = lambda *s: (torch.rand(*s, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)  # noqa: E731
        kp, vp = rnd(prefix, hkv, 128), rnd(prefix, hkv, 128)
        root = st.create()
        st.append_many(root, torch.full((prefix,), 11, dtype=torch.int32, device="cuda"),
                       torch.arange(prefix, dtype=torch.int32, device="cuda"), 0, kp, vp)
        kids = st.fork(root, B)
        st.release(root)
        for bi, h in enumerate(kids):
            kb, vb = rnd(blen - 1, hkv, 128), rnd(blen - 1, hkv, 128)
            st.append_many(h, torch.full((blen - 1,), 12, dtype=torch.int32, device="cuda"),
                           torch.arange(prefix, prefix + blen - 1, dtype=torch.int32, device="cuda"), 0, kb, vb)
            if bi in sample.get(r, []):
                kept[(r, bi)] = (kp.cpu(), vp.cpu(), kb.cpu(), vb.cpu(), len(handles))
            handles.append(h)
            qpos.append(prefix + blen - 1)
    n = len(handles)
    knew, vnew, q = sym_bf16(31, (n, hkv, 128)), sym_bf16(32, (n, hkv, 128)), sym_bf16(33, (n, hq, 128))
    pos = torch.tensor(qpos, dtype=torch.int32)
    st.append(handles, torch.full((n,), 13, dtype=torch.int32, device="cuda"), pos.cuda(), 0, knew.cuda(), vnew.cuda())
    out = mv.attention.decode(st, handles, q.cuda(), pos.cuda(), out_dtype=torch.float32)
    torch.cuda.synchronize()
    info = st.plan_info()
    assert info["unique_kv_tokens"] == R * (prefix + B * blen)
    o = out.cpu().numpy()
    assert np.isfinite(o).all()
    for (r, bi), (kp, vp, kb, vb, idx) in kept.items():
        K = np.concatenate([bf16_to_f64(kp), bf16_to_f64(kb), bf16_to_f64(knew[idx:idx + 1])])
        V = np.concatenate([bf16_to_f64(vp), bf16_to_f64(vb), bf16_to_f64(vnew[idx:idx + 1])])
        P = np.concatenate([np.arange(prefix), np.arange(prefix, prefix + blen - 1), [qpos[idx]]]).astype(np.int32)
        ref = oracle.attn_decode(oracle.rope(bf16_to_f64(q[idx:idx + 1]), pos[idx:idx + 1].numpy()), oracle.rope(K, P), V,
                                 [list(range(len(P)))])
        err = np.abs(o[idx:idx + 1] - ref).max()
        assert err < TOL, ((r, bi), err)


def test_c5_reduce_merge_full_scale(mv):
    """BASELINE configs[4] at full size: 4,096-token prefix, 16 rounds of {fork 128; append 64
    tokens per branch; zero-copy merge in ordinal order; append 16 Reduce tokens}, then decode
    steps over the merged 135,424-token context.  Every fork / merge moves 0 KV bytes and
    allocates no page; the final decode matches the oracle."""
    hq, hkv, B, rounds, path, red, prefix = 40, 8, 128, 16, 64, 16, 4096
    total = prefix + rounds * (B * path + red)
    assert total == 135424
    pages = total // 16 + rounds * B * 2 + 4096
    # every fork gives each of the 128 children its own copy of the parent's span list (as the
    # reference does, kvcache.cpp:245-252): ~2 x 128 x 8.5K entries in the last round
    st = mv.kv.PagedStore(num_pages=pages, layers=1, kv_heads=hkv, table_entries=1 << 23)
    g = torch.Generator(device="cuda")
    g.manual_seed(555)
    ks, vs, ps = [], [], []

    def add(h, n, pos0):
        k = (torch.rand(n, hkv, 128, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
        v = (torch.rand(n, hkv, 128, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
        p = torch.arange(pos0, pos0 + n, dtype=torch.int32, device="cuda")
        st.append_many(h, torch.full((n,), 11, dtype=torch.int32, device="cuda"), p, 0, k, v)
        ks.append(k)
        vs.append(v)
        ps.append(p)

    cur = st.create()
    add(cur, prefix, 0)
    L = prefix
    for _ in range(rounds):
        kids = st.fork(cur, B)
        assert st.stats().bytes_copied_on_last_op == 0
        for k in kids:
            add(k, path, L)  # siblings share their start position
        free_before = st.stats().free_pages
        m = st.merge(cur, kids)
        s = st.stats()
        assert s.bytes_copied_on_last_op == 0 and s.free_pages == free_before
        for h in [cur] + kids:
            st.release(h)
        L += path
        add(m, red, L)
        L += red
        cur = m
    assert st.length(cur) == total
    for step in range(4):
        kn, vn = sym_bf16(8800 + step, (1, hkv, 128)), sym_bf16(8900 + step, (1, hkv, 128))
        q = sym_bf16(9900 + step, (1, hq, 128))
        pos = torch.tensor([L], dtype=torch.int32)
        st.append([cur], torch.tensor([13], dtype=torch.int32, device="cuda"), pos.cuda(), 0, kn.cuda(), vn.cuda())
        ks.append(kn.cuda())
        vs.append(vn.cuda())
        ps.append(pos.cuda())
        out = mv.attention.decode(st, [cur], q.cuda(), pos.cuda(), out_dtype=torch.float32)
        L += 1
    K = bf16_to_f64(torch.cat(ks).cpu())
    V = bf16_to_f64(torch.cat(vs).cpu())
    P = torch.cat(ps).cpu().numpy()
    ref = oracle.attn_decode(oracle.rope(bf16_to_f64(q), pos.numpy()), oracle.rope(K, P), V, [list(range(len(P)))])
    assert np.abs(out.float().cpu().numpy() - ref).max() < TOL
    st.release(cur)
    s = st.stats()
    assert s.live_handles == 0 and s.total_refcount == 0 and s.free_pages == pages


@pytest.mark.parametrize("hq,hkv,branches", [(40, 1, 3), (8, 8, 5), (16, 4, 9), (32, 8, 12)])
def test_gqa_and_copy_layouts(mv, hq, hkv, branches):
    """Row layouts across GQA ratios: one KV head with 40 query heads (64-row members), MHA,
    and member counts that make 33-64-row cascade units (planned with a second row copy) and
    > 64-row units."""
    err, _ = run_case(mv, [(200, branches, 45)], hq=hq, hkv=hkv, num_pages=512, seed=hq + branches)
    assert err < TOL, err


def test_row_copy_layouts_after_plain_units(mv):
    """Long private chunks (1 member, plain layout) are scheduled before short cascade chunks of
    6 members (48 rows: planned with row copies), so CTAs switch from plain to copied units
    while some softmax warps of the previous unit are still running."""
    err, st = run_case(mv, [(64, 6, 1500)] * 6, hq=40, hkv=8, num_pages=8192, seed=77)
    assert err < TOL, err
    assert st.plan_info()["work_items"] >= 6 * 7


def test_device_produced_inputs_without_sync(mv):
    """Engine-style stream ordering: every step's K/V, positions and queries are written by a
    device kernel into the SAME buffers right before the append / decode that read them (holding
    the previous step's values until then), behind a long GEMM, with no host synchronisation
    across 12 steps.  The append, the RoPE pre-pass and decode_tc are launched programmatically
    dependent (PDL): a read issued ahead of its griddepcontrol.wait would see the stale values."""
    hq, hkv, steps = 40, 8, 12
    st = mv.kv.PagedStore(num_pages=512, layers=1, kv_heads=hkv)
    rows = {"k": [], "v": [], "pos": []}
    r = Req(mv, st, rows, 21, 300, 4, 40, hkv=hkv)
    handles, ctx, qpos = list(r.handles), [list(c) for c in r.ctx], list(r.qpos)
    n = len(handles)
    ks = [sym_bf16(7000 + s * 3, (n, hkv, 128)) for s in range(steps)]
    vs = [sym_bf16(7001 + s * 3, (n, hkv, 128)) for s in range(steps)]
    qs = [sym_bf16(7002 + s * 3, (n, hq, 128)) for s in range(steps)]
    ks_d, vs_d, qs_d = [x.cuda() for x in ks], [x.cuda() for x in vs], [x.cuda() for x in qs]
    kbuf, vbuf, qbuf = torch.empty_like(ks_d[0]), torch.empty_like(vs_d[0]), torch.empty_like(qs_d[0])
    pbuf = torch.tensor(qpos, dtype=torch.int32, device="cuda") - 1
    toks = torch.full((n,), 12, dtype=torch.int32, device="cuda")
    big = torch.randn(4096, 4096, dtype=torch.bfloat16, device="cuda")
    outs = []
    torch.cuda.synchronize()
    for s in range(steps):
        _ = big @ big  # keeps the GPU busy so PDL launches start early
        torch.add(pbuf, 1, out=pbuf)
        torch.mul(ks_d[s], 1, out=kbuf)
        torch.mul(vs_d[s], 1, out=vbuf)
        st.append(handles, toks, pbuf, 0, kbuf, vbuf)
        _ = big @ big
        torch.mul(qs_d[s], 1, out=qbuf)
        outs.append(mv.attention.decode(st, handles, qbuf, pbuf, out_dtype=torch.float32))
    torch.cuda.synchronize()
    for s in range(steps):
        pos = torch.tensor([p + s for p in qpos], dtype=torch.int32)
        base = sum(x.shape[0] for x in rows["k"])
        rows["k"].append(ks[s])
        rows["v"].append(vs[s])
        rows["pos"].append(pos)
        for i in range(n):
            ctx[i].append(base + i)
        K = np.concatenate([bf16_to_f64(x) for x in rows["k"]])
        V = np.concatenate([bf16_to_f64(x) for x in rows["v"]])
        P = np.concatenate([x.numpy() for x in rows["pos"]])
        ref = oracle.attn_decode(oracle.rope(bf16_to_f64(qs[s]), pos.numpy()), oracle.rope(K, P), V, ctx)
        err = np.abs(outs[s].cpu().numpy() - ref).max()
        assert err < TOL, (s, err)


# ---- head dim 64 (the toy model's d_h, toy_model.hpp:29): native decode_tc_kernel<64> ----
@pytest.mark.parametrize("spec,hq,hkv", [
    ([(100, 3, 20)], 40, 8),                          # plain units, ragged pages
    ([(1000, 8, 300), (64, 2, 17)], 40, 8),           # F = 2 row copies (8 x 5 rows)
    ([(4096, 32, 100)], 40, 8),                       # > 16 members: member groups
    ([(16, 1, 9000)], 40, 8),                         # split-KV slots + combine
    ([(333, 4, 70), (50, 2, 5, (20, 3))], 4, 4),      # MHA (C1's 4 heads), nested lineage
])
def test_head_dim_64(mv, spec, hq, hkv):
    err, _ = run_case(mv, spec, hq, hkv, 4096, seed=11, d=64)
    assert err < TOL


def test_head_dim_64_score_spike(mv):
    err, _ = run_case(mv, [(300, 4, 40)], 40, 8, 512, seed=12, spike=True, d=64)
    assert err < TOL


def test_head_dim_mismatch_raises(mv):
    st = mv.kv.PagedStore(num_pages=16, layers=1, kv_heads=2, head_dim=64)
    h = st.create()
    k = sym_bf16(1, (3, 2, 64)).cuda()
    st.append_many(h, torch.full((3,), 11, dtype=torch.int32, device="cuda"),
                   torch.arange(3, dtype=torch.int32, device="cuda"), 0, k, k)
    with pytest.raises(ValueError):
        mv.attention.decode(st, [h], sym_bf16(2, (1, 4, 128)).cuda(), torch.tensor([3], dtype=torch.int32).cuda())
    with pytest.raises(ValueError):  # MV_ERR_INVALID_ARGUMENT: no kernel for head dim 96
        mv.kv.PagedStore(num_pages=16, layers=1, kv_heads=2, head_dim=96)


def test_decode_kernel_timing_hook(mv):
    """mv_attn_decode_kernel_timing records one event pair per decode_tc launch (bench.py's roofline timing):
    as many durations as recorded calls, each positive, and recording off once re-armed with 0."""
    err, st = run_case(mv, [(300, 3, 37)], hq=8, hkv=2, num_pages=256)
    st.decode_kernel_timing(4)
    assert st.decode_kernel_timing(4) == []  # nothing recorded yet
    h = st.create()
    k = sym_bf16(5, (40, 2, 128)).cuda()
    st.append_many(h, torch.full((40,), 11, dtype=torch.int32, device="cuda"),
                   torch.arange(40, dtype=torch.int32, device="cuda"), 0, k, k)
    q = sym_bf16(6, (1, 8, 128)).cuda()
    p = torch.tensor([40], dtype=torch.int32, device="cuda")
    for _ in range(3):
        mv.attention.decode(st, [h], q, p)
    ms = st.decode_kernel_timing(0)
    assert len(ms) == 3 and all(0.0 < x < 100.0 for x in ms)
    mv.attention.decode(st, [h], q, p)
    assert st.decode_kernel_timing(0) == []
