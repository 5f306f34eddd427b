"""Per-op parity of the sm_100a kernels against the oracle (run on a B200).

Tolerances: integer / index work bit-exact; attention
fp32 output <= 6e-3 max-abs (P is rounded to bf16 for the PV tensor-core product:
|do| <= 2^-9 max|v|, ~2.4e-3 observed for N(0,1) values; inside the 1e-2 contract); bf16 outputs <= 1e-2 + 1 bf16 ulp of the
value; GEMM fp32 partials vs fp64 on the same bf16 inputs <= 1e-3 * sqrt(K)-scaled.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import weights as OW                      # noqa: E402
from oracle.model import paged_attention as o_attn   # noqa: E402
from oracle.priority import priority as o_priority   # noqa: E402
from oracle.merge import merge_rank_topk            # noqa: E402


@pytest.fixture(scope="module")
def rt():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2412_18695_b200 import rt as _rt
    _rt.lib()
    return _rt


def bf16_t(a):
    return torch.from_numpy(np.asarray(a, dtype=np.float32)).to(torch.bfloat16)


@pytest.mark.parametrize("tid,n", [(0, 4096 * 3 + 17), (1, 100000), (16 + 8 * 3 + 2, 65536)])
def test_init_weights_bitexact(rt, tid, n):
    out = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    rt.init_weights(out, n, 0xC0FFEE, tid, 0.02)
    torch.cuda.synchronize()
    got = out.view(torch.int16).cpu().numpy().view(np.uint16)
    ref = OW.weight_values(0xC0FFEE, tid, np.arange(n, dtype=np.uint64), 0.02)
    refb = (ref.view(np.uint32) >> 16).astype(np.uint16)
    assert np.array_equal(got, refb)


def test_priority_bitexact(rt):
    rng = np.random.default_rng(0)
    n = 5000
    t = rng.integers(0, 5_000_000, n)
    ref_ = t - rng.integers(-3_000_000, 2_000_000, n)
    D = t + rng.integers(-2_000_000, 3_000_000, n)
    ert = rng.integers(0, 2_000_000, n)
    k = rng.integers(0, 3, n).astype(np.int32)
    alpha = -rng.uniform(0, 10, n)
    alpha[::7] = -6.67
    beta = rng.uniform(-2, 3, n)
    beta[::11] = 0.0
    trde = np.stack([t, ref_, D, ert], axis=1).astype(np.int64)
    dt = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    rt.priority(dt(trde), dt(k), dt(alpha), dt(beta), 90000, 8000, 1000, out)
    got = out.cpu().numpy()
    ref = np.array([o_priority(int(t[i]), int(k[i]), int(ref_[i]), int(D[i]), int(ert[i]), float(alpha[i]),
                               float(beta[i]), 90000, 8000, 1000) for i in range(n)])
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("M,N,K,splits", [(256, 64, 512, 1), (384, 7, 1024, 4), (200, 130, 256, 2),
                                          (6144, 64, 4096, 6), (1024, 300, 768, 1), (512, 32, 14336, 8),
                                          (4096, 64, 4096, 9), (1024, 64, 14336, 16), (640, 100, 2048, 3),
                                          (384, 150, 512, 1), (384, 190, 768, 2), (512, 350, 512, 1),
                                          (256, 470, 1024, 3), (6144, 161, 4096, 0),
                                          (19200, 200, 512, 0), (20480, 150, 1024, 0), (9728, 300, 512, 0),
                                          (28672, 320, 512, 0), (38400, 150, 256, 0)])
def test_gemm_tcgen05(rt, M, N, K, splits):
    g = torch.Generator().manual_seed(M * 7 + N)
    W = (torch.randn(M, K, generator=g) * 0.05).to(torch.bfloat16)
    n_cap = ((N + 255) // 256) * 256
    X = torch.zeros(n_cap, K, dtype=torch.bfloat16)
    X[:N] = torch.randn(N, K, generator=g).to(torch.bfloat16)
    Wd, Xd = W.cuda(), X.cuda()
    out = torch.full((N, M), float("nan"), device="cuda")
    rt.gemm(Wd, Xd, out, M, N, K, n_cap, splits)
    torch.cuda.synchronize()
    got = out.double().cpu()
    ref = X[:N].double() @ W.double().T
    err = (got - ref).abs().max().item()
    assert err < 1e-3 * max(1.0, (K / 512) ** 0.5), err


def _gemm_tiled_case(rt, M, N, K, path, bn=0, splits=0):
    """The engine's layout (rt_op_pack_tiled) through one forced kernel path, vs fp64."""
    g = torch.Generator().manual_seed(M * 7 + N + path)
    W = (torch.randn(M, K, generator=g) * 0.05).to(torch.bfloat16)
    n_cap = ((N + 255) // 256) * 256
    X = torch.zeros(n_cap, K, dtype=torch.bfloat16)
    X[:N] = torch.randn(N, K, generator=g).to(torch.bfloat16)
    Wd, Xd = W.cuda(), X.cuda()
    Wt = torch.zeros(((M + 127) // 128) * 128 * K, dtype=torch.bfloat16, device="cuda")
    rt.pack_tiled(Wd, Wt, M, K)
    out = torch.full((N, M), float("nan"), device="cuda")
    rt.gemm_tiled(Wt, Xd, out, M, N, K, n_cap, splits, path=path, bn=bn)
    torch.cuda.synchronize()
    ref = X[:N].double() @ W.double().T
    err = (out.double().cpu() - ref).abs().max().item()
    assert err < 1e-3 * max(1.0, (K / 512) ** 0.5), err


@pytest.mark.parametrize("M,N,K", [(28672, 320, 512), (28672, 512, 4096), (19200, 200, 512), (38400, 150, 256),
                                   (9728, 300, 512), (20480, 161, 1024), (6144, 1600, 1024), (4096, 1600, 2048),
                                   (6144, 256, 4096), (512, 200, 256)])
def test_gemm_cta_pair(rt, M, N, K):
    """CTA-pair projections (tcgen05.mma.cta_group::2, RT_GEMM_PATH_PAIR): N > 128 and an even
    number of 128-row m-tiles; ragged N (161, 200, 300) leaves the second CTA's half of the last
    n-tile partly empty; fewer pair-tiles than co-resident pairs (6144 x 256, 512 x 200) and a
    partial last round (sub-tiles) are covered."""
    assert (M // 128) % 2 == 0
    _gemm_tiled_case(rt, M, N, K, rt.RT_GEMM_PATH_PAIR)


@pytest.mark.parametrize("M,N,K,bn", [(28672, 512, 512, 256), (9728, 1024, 512, 0), (6144, 1600, 1024, 160),
                                      (4096, 1600, 2048, 192), (28672, 330, 768, 160)])
def test_gemm_streamk(rt, M, N, K, bn):
    """Hybrid data-parallel + stream-K (k_gemm_sk, more than two waves of tiles: the full waves
    but one data-parallel, the rest stream-K with multi-contributor fixups), CTA pairs excluded."""
    _gemm_tiled_case(rt, M, N, K, rt.RT_GEMM_PATH_STREAMK, bn=bn)


@pytest.mark.parametrize("M,N,K", [(6144, 256, 4096), (4096, 256, 4096), (4096, 256, 14336), (6144, 200, 4096),
                                   (4096, 64, 4096), (6144, 33, 1024), (512, 129, 512), (4096, 128, 14336),
                                   (8192, 256, 8192), (10240, 256, 8192)])
def test_gemm_decode_pair_splitk(rt, M, N, K):
    """k_gemm_dec (RT_GEMM_PATH_DECPAIR): CTA pairs (cta_group::2, M = 256) with a cluster split-K
    over pairs and the DSMEM reduction, at the 8B / 70B decode shapes (QKV 6144 / 10240, O and
    down 4096 / 8192 rows) and ragged batches (33, 129, 200 rows)."""
    _gemm_tiled_case(rt, M, N, K, 4)


@pytest.mark.parametrize("M,N,K,bn", [(28672, 256, 512, 256), (6144, 200, 1024, 0), (4096, 384, 2048, 192)])
def test_gemm_splitk_wide(rt, M, N, K, bn):
    """k_gemm_tc forced on prefill-sized N (one tile per CTA / wave-tail split)."""
    _gemm_tiled_case(rt, M, N, K, rt.RT_GEMM_PATH_SPLITK, bn=bn)


@pytest.mark.parametrize("M,N,K", [(512, 4, 128), (128256, 64, 1024), (1000, 33, 256), (128256, 256, 1024),
                                   (20480, 200, 512)])
def test_lm_argmax(rt, M, N, K):
    g = torch.Generator().manual_seed(N)
    W = (torch.randn(M, K, generator=g) * 0.02).to(torch.bfloat16)
    X = torch.randn(N, K, generator=g).to(torch.bfloat16)
    tok = torch.empty(N, dtype=torch.int32, device="cuda")
    logits = torch.empty(N, M, device="cuda")
    rt.lm_argmax(W.cuda(), X.cuda().contiguous(), M, N, K, N, tok, logits)
    torch.cuda.synchronize()
    ref = X.double() @ W.double().T
    assert (logits.double().cpu() - ref).abs().max().item() < 1e-3
    lg = logits.cpu().numpy()
    assert np.array_equal(tok.cpu().numpy(), np.argmax(lg, axis=1))   # lowest index on ties


def _attn_case(rt, hd, nq, nkv, seqlens, seed, n_pages=None, f32=True):
    rng = np.random.default_rng(seed)
    P = 16
    max_pages = max((s + P - 1) // P for s in seqlens)
    need = sum((s + P - 1) // P for s in seqlens)
    n_pages = n_pages or need + 5
    perm = rng.permutation(n_pages)
    tables, used = [], 0
    for s in seqlens:
        k = (s + P - 1) // P
        tables.append(list(perm[used:used + k]) + [0] * (max_pages - k))
        used += k
    # random logical K/V for every (page, slot) -> write through rt_op_kv_write
    kv_k = bf16_t(rng.standard_normal((n_pages * P, nkv, hd)))
    kv_v = bf16_t(rng.standard_normal((n_pages * P, nkv, hd)))
    pool = torch.zeros(n_pages * nkv * 64 * hd, dtype=torch.uint8, device="cuda")
    slots = torch.arange(n_pages * P, dtype=torch.int32, device="cuda")
    rt.kv_write(pool, kv_k.cuda(), kv_v.cuda(), slots, nkv, hd)
    q = bf16_t(rng.standard_normal((len(seqlens), nq, hd)))
    pt = torch.tensor(np.array(tables, dtype=np.int32)).cuda()
    row_task = torch.arange(len(seqlens), dtype=torch.int32, device="cuda")
    row_sl = torch.tensor(seqlens, dtype=torch.int32, device="cuda")
    out = torch.empty(len(seqlens), nq, hd, dtype=torch.bfloat16, device="cuda")
    out32 = torch.empty(len(seqlens), nq, hd, device="cuda") if f32 else None
    rt.paged_attention(q.cuda(), pool, pt, row_task, row_sl, max(seqlens), nq, nkv, hd, out, out32)
    torch.cuda.synchronize()
    kp = kv_k.float().numpy().reshape(n_pages, P, nkv, hd)
    vp = kv_v.float().numpy().reshape(n_pages, P, nkv, hd)
    qf = q.float().numpy()
    errs32, errs16 = [], []
    for r, s in enumerate(seqlens):
        ref = o_attn(qf[r], kp, vp, tables[r], s, P)
        got16 = out[r].float().cpu().numpy()
        tol16 = 1e-2 + np.abs(ref) * 2.0 ** -8
        errs16.append(float(np.max(np.abs(got16 - ref) - tol16)))
        if f32:
            errs32.append(float(np.max(np.abs(out32[r].cpu().numpy() - ref))))
    # read-back of the pool is the identity on the logical layout
    back = torch.empty(n_pages, 2, nkv, P, hd, dtype=torch.bfloat16, device="cuda")
    rt.kv_read(pool, back, n_pages, nkv, hd)
    b = back.cpu()
    assert torch.equal(b[:, 0].permute(0, 2, 1, 3).reshape(-1, nkv, hd), kv_k)
    assert torch.equal(b[:, 1].permute(0, 2, 1, 3).reshape(-1, nkv, hd), kv_v)
    return max(errs32) if f32 else 0.0, max(errs16)


@pytest.mark.parametrize("hd,nq,nkv", [(128, 32, 8), (128, 64, 8), (32, 4, 1), (64, 8, 2), (128, 8, 8)])
def test_paged_attention_ragged(rt, hd, nq, nkv):
    seqlens = [1, 15, 16, 17, 33, 100, 257, 1310]
    e32, e16 = _attn_case(rt, hd, nq, nkv, seqlens, seed=hd + nq)
    assert e32 < 6e-3, e32
    assert e16 <= 0.0, e16


def test_paged_attention_split_kv_long(rt):
    # few rows, long contexts -> split-KV chunks + combine kernel
    e32, e16 = _attn_case(rt, 128, 32, 8, [8192, 2884, 4000], seed=3)
    assert e32 < 6e-3 and e16 <= 0.0


def test_paged_attention_c2_operating_point_sampled(rt):
    # 64 rows at ctx 1310 (C2), 8B heads; all rows checked (cheap in numpy)
    e32, e16 = _attn_case(rt, 128, 32, 8, [1310] * 64, seed=9)
    assert e32 < 6e-3 and e16 <= 0.0


def test_kv_swap_roundtrip(rt):
    """rt_op_kv_swap (R-EVICT copies): pages evicted to pinned host pages and restored into
    different device pages are bit-identical, every layer, untouched pages unchanged."""
    L, n_pages, nkv, hd = 3, 12, 2, 64
    blk = nkv * 2 * 16 * hd * 2
    g = torch.Generator(device="cuda").manual_seed(0)
    pool = torch.randint(0, 255, (L, n_pages * blk), dtype=torch.uint8, device="cuda", generator=g)
    orig = pool.clone()
    host = torch.zeros(8 * L * blk, dtype=torch.uint8).pin_memory()
    ev = torch.tensor([[0, 0, 3, 5], [0, 0, 7, 0], [0, 1, 1, 2]], dtype=torch.int32, device="cuda")
    rt.kv_swap(ev, pool, n_pages * blk, host, blk, L)
    torch.cuda.synchronize()
    hv = host.view(8, L, blk)
    for _, _, dp, hp in ev.tolist():
        for l in range(L):
            assert torch.equal(hv[hp, l].cuda(), orig[l, dp * blk:(dp + 1) * blk])
    rs = torch.tensor([[1, 0, 10, 5], [1, 0, 11, 0], [1, 1, 4, 2]], dtype=torch.int32, device="cuda")
    rt.kv_swap(rs, pool, n_pages * blk, host, blk, L)
    torch.cuda.synchronize()
    for (_, _, src, _), (_, _, dst, _) in zip(ev.tolist(), rs.tolist()):
        assert torch.equal(pool[:, dst * blk:(dst + 1) * blk], orig[:, src * blk:(src + 1) * blk])
    keep = [p for p in range(n_pages) if p not in (10, 11, 4)]
    for p in keep:
        assert torch.equal(pool[:, p * blk:(p + 1) * blk], orig[:, p * blk:(p + 1) * blk])


@pytest.mark.parametrize("world", [1, 2, 3, 5, 8])
def test_merge_candidates_matches_oracle(rt, world):
    """a12 device merge (rt_op_merge_candidates, the kernel every rank runs on the allgathered
    candidates) against oracle c13 on G synthetic rank buffers: per-rank top-16 lists sorted by
    (Pri desc, arrival asc, id asc) with ties in Pri and in (Pri, arrival) across ranks, empty
    slots (rid -1) at the end of short lists, and -0.0 canonicalised upstream."""
    K = 16
    for trial in range(20):
        rng = np.random.default_rng(world * 100 + trial)
        lists, rid = [], 0
        for r in range(world):
            n = int(rng.integers(0, K + 1)) if trial % 3 else K
            pri = rng.choice([13.7174, 15.6495, 202.02, -4400.0, 1.0], size=n) if trial % 2 else rng.normal(0, 50, n)
            arr = rng.choice([0, 100000, 200000], size=n) if trial % 2 else rng.integers(0, 10 ** 7, n)
            recs = []
            for i in range(n):
                recs.append((float(pri[i]), float(arr[i]), float(rid * world + r), float(r)))
                rid += 1
            recs.sort(key=lambda x: (-x[0], x[1], x[2]))
            lists.append(recs)
        buf = np.zeros((world, K, 4))
        buf[:, :, 2] = -1.0
        for r, recs in enumerate(lists):
            if recs:
                buf[r, :len(recs)] = np.array(recs)
        d_all = torch.from_numpy(buf).cuda()
        merged = torch.full((K, 4), float("nan"), dtype=torch.float64, device="cuda")
        rt.merge_candidates(d_all, world, merged)
        torch.cuda.synchronize()
        got = merged.cpu().numpy()
        ref = merge_rank_topk(lists, K)
        n_valid = len(ref)
        assert np.array_equal(got[:n_valid], np.array(ref).reshape(n_valid, 4)), (world, trial)
        assert (got[n_valid:, 2] < 0).all()


@pytest.mark.parametrize("hd,nq,nkv,groups", [(128, 32, 8, 0), (128, 32, 8, 1), (128, 32, 8, 2), (128, 64, 8, 1),
                                              (64, 16, 4, 2), (64, 16, 2, 1), (32, 4, 1, 0)])
def test_prefill_attention_causal(rt, hd, nq, nkv, groups):
    """k_attn_prefill (rt_op_prefill_attention) per causal row against oracle.paged_attention:
    prompt lengths 1 .. 2884 (PAPER.md:71 arm prompt), prompt rows starting at a prefix offset
    pos0 > 0 (shared-prefix tails, R-PFX: 1216 = 76 pages) and at 0, ragged last tiles,
    G = 1 / 2 / 4 / 8, one and two warp groups; rows sampled for the long prompts (every tile's
    first and last row, the rows around each page boundary)."""
    rng = np.random.default_rng(hd * 7 + nq + groups)
    P = 16
    # (prompt length, first prompt row position): tail prefill after a shared prefix or whole prompt
    cases = [(1, 0), (15, 0), (17, 0), (100, 0), (1300, 1216), (2884, 2800), (1300, 0), (40, 32)]
    if hd == 32:
        cases = [(1, 0), (17, 0), (100, 0), (300, 256)]
    max_pages = max((L + P - 1) // P for L, _ in cases)
    n_pages = sum((L + P - 1) // P for L, _ in cases) + 3
    perm = rng.permutation(n_pages)
    tables, used = [], 0
    for L, _ in cases:
        k = (L + P - 1) // P
        tables.append(list(perm[used:used + k]) + [0] * (max_pages - k))
        used += k
    kv_k = bf16_t(rng.standard_normal((n_pages * P, nkv, hd)))
    kv_v = bf16_t(rng.standard_normal((n_pages * P, nkv, hd)))
    pool = torch.zeros(n_pages * nkv * 64 * hd, dtype=torch.uint8, device="cuda")
    rt.kv_write(pool, kv_k.cuda(), kv_v.cuda(), torch.arange(n_pages * P, dtype=torch.int32, device="cuda"), nkv, hd)
    rows, tiles = [], []
    for t, (L, start) in enumerate(cases):
        for pos0 in range(start - start % P, L, P):
            lo = max(pos0, start)
            hi = min(pos0 + P, L)
            # a tile's rows are consecutive positions pos0 + i; the first tile of a tail may start
            # mid-page only when start is not page aligned (never here: prefixes are whole pages)
            assert lo == pos0
            tiles.append((len(rows), hi - lo, pos0, t))
            rows += [(t, p) for p in range(lo, hi)]
    q = bf16_t(rng.standard_normal((len(rows), nq, hd)))
    out = torch.empty(len(rows), nq, hd, dtype=torch.bfloat16, device="cuda")
    out32 = torch.full((len(rows), nq, hd), float("nan"), device="cuda")
    pt = torch.tensor(np.array(tables, dtype=np.int32)).cuda()
    tl = torch.tensor(np.array(tiles, dtype=np.int32)).cuda()
    rt.prefill_attention(q.cuda(), pool, pt, tl, nq, nkv, hd, out, out32, groups=groups)
    torch.cuda.synchronize()
    kp = kv_k.float().numpy().reshape(n_pages, P, nkv, hd)
    vp = kv_v.float().numpy().reshape(n_pages, P, nkv, hd)
    o32 = out32.cpu().numpy()
    ob = out.float().cpu().numpy()
    qn = q.float().numpy()
    sample = set()
    for (r0, nr, pos0, t) in tiles:
        sample.update({r0, r0 + nr - 1, r0 + nr // 2})
    sample.update(int(x) for x in rng.choice(len(rows), size=min(len(rows), 48), replace=False))
    worst = worst_b = 0.0
    for i in sorted(sample):
        t, p = rows[i]
        ref = o_attn(qn[i], kp, vp, tables[t], p + 1)
        worst = max(worst, float(np.abs(o32[i] - ref).max()))
        worst_b = max(worst_b, float((np.abs(ob[i] - ref) - np.abs(ref) * 2.0 ** -8).max()))
    # the 1e-2 contract (BASELINE.json): P is rounded to bf16 for the P.V tensor-core product,
    # |dP| <= u P with u = 2^-8, so |do| <= u max|v| ~ 0.4 * 2^-8 * 4; short prompts (a few
    # positions) do not average it out (observed ~8e-3 at 1..17 positions)
    assert worst < 1e-2, worst
    assert worst_b < 1e-2, worst_b
