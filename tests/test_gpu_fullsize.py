"""Full-size per-op oracle parity of the decode layer (Llama-3-8B and -70B layer dims).

The graded step runs the fused tcgen05 epilogues at d = 4096 / 8192, hd = 128 with 8 kv heads.
These tests run the engine at those dims (2 layers, full vocabulary) on the workload's shapes —
64 decode rows at contexts >= 1300 (drone prompts) and a prefill round of >= 512
prompt rows made of shared-prefix tails (R-PFX) — and check EVERY fused output of
every layer against oracle ops applied to the GPU's own inputs (AMB-16: per op on identical
inputs), from the per-layer captures (RT_FLAG_CAPTURE_LAYERS):

  QKV + RoPE        q  = bf16(rope(bf16(rms(x)) W_q^T))           vs the GPU's q        (sampled heads)
  KV append         k  = bf16(rope(bf16(rms(x)) W_k^T)), v = bf16(bf16(rms(x)) W_v^T)
                                                                   vs the layer's pages at (task, pos)
  attention         o  = paged_attention(GPU q, GPU pages)        vs the GPU's o        (sampled rows)
  O + residual      x' = x + o W_o^T                              vs the GPU's x after O
  gate/up + SwiGLU  a  = bf16(silu(h W_g^T) * (h W_u^T)), h = bf16(rms(x'))
                                                                   vs the GPU's activation
  down + residual   x'' = x' + a W_d^T                            vs the GPU's next-layer input

Output features are sampled (whole heads for q/k/v, random rows of W_o / W_gate_up / W_down:
the oracle regenerates only those weight rows from the counter-based init) — every row of the
round is checked on them.  Tolerances (DESIGN.md §4 / R-NORM): bf16 outputs within 1e-2 + one
bf16 ulp of the value + the R-NORM shift of that element (the GPU rounds x, not rms(x), to
bf16: the exact difference of the two operands, projected through the element's weight row,
computed from the GPU's own x); fp32 residual outputs within 1e-3 sqrt(K / 512) (fp32 vs fp64
accumulation of identical bf16 operands).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import weights as OW                                     # noqa: E402
from oracle.bf16 import bf16                                         # noqa: E402
from oracle.model import rms, rope, silu, paged_attention            # noqa: E402
from synth import MODEL_SHAPES, make_vocab, engine_params            # noqa: E402
from synth.configs import ModelShape                                 # noqa: E402
from synth.traces import make_trace, system_prefix                   # noqa: E402


@pytest.fixture(scope="module")
def rt():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2412_18695_b200 import rt as _rt
    _rt.lib()
    return _rt


def bf(u16):
    return (np.asarray(u16, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def ulp_tol(ref):
    """1e-2 + one bf16 ulp of the value (both sides round to bf16 at the same point)."""
    return 1e-2 + np.abs(ref) * 2.0 ** -7


class Checker:
    def __init__(self, shape, seed):
        self.s, self.seed = shape, seed
        self.worst = {}

    def note(self, key, err):
        self.worst[key] = max(self.worst.get(key, 0.0), float(err))

    def W(self, l, j, rows, n_in):
        return OW.matrix(self.seed, OW.layer_tid(l, j), np.asarray(rows, dtype=np.uint64), n_in)

    def layer(self, eng, rt, l, rows, tabs, rng, attn_rows):
        s = self.s
        d, nq, nkv, hd, ff = s.d_model, s.n_q_heads, s.n_kv_heads, s.head_dim, s.d_ff
        n = len(rows)
        x = eng.layer_dump(rt.RT_DUMP_LAYER_X, l, np.float32).reshape(n, d).astype(np.float64)
        q = bf(eng.layer_dump(rt.RT_DUMP_LAYER_Q, l, np.uint16)).reshape(n, nq, hd)
        o = bf(eng.layer_dump(rt.RT_DUMP_LAYER_O, l, np.uint16)).reshape(n, nq, hd)
        xm = eng.layer_dump(rt.RT_DUMP_LAYER_XMID, l, np.float32).reshape(n, d).astype(np.float64)
        act = bf(eng.layer_dump(rt.RT_DUMP_LAYER_ACT, l, np.uint16)).reshape(n, ff)
        xo = eng.layer_dump(rt.RT_DUMP_LAYER_X, l + 1, np.float32).reshape(n, d).astype(np.float64)
        kv = eng.layer_dump(rt.RT_DUMP_LAYER_KV, l, np.uint16).reshape(-1, 2, nkv, 16, hd)   # raw bf16 bits
        pos = np.array([r[1] for r in rows])
        task = np.array([r[0] for r in rows])
        # ---- QKV + RoPE + KV append (sampled heads: 2 q heads, 2 k heads, 2 v heads)
        # reading R-NORM: the GPU rounds x (not rms(x)) to bf16 and applies the row scale in the
        # epilogue; the shift this moves into each output is computed exactly from the GPU's x
        # and added to the tolerance (1e-2 + one bf16 ulp + |R-NORM shift|)
        h = bf16(rms(x))
        hs = bf16(x) / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + 1e-5)   # the GPU's operand x scale
        dh = hs - h
        qh = sorted({0, int(rng.integers(1, nq))})
        kh = sorted({0, int(rng.integers(1, nkv))})

        def rope_shift(wrows):   # |rope(shift)| <= |shift_i| + |shift_{i + hd/2}| in both halves
            sh = dh @ wrows.T
            b = np.abs(sh[:, :hd // 2]) + np.abs(sh[:, hd // 2:])
            return np.concatenate([b, b], axis=-1)

        for hq in qh:
            wq = self.W(l, OW.TID_QKV, range(hq * hd, (hq + 1) * hd), d)
            ref = bf16(rope((h @ wq.T)[:, None, :], pos, hd)[:, 0])
            tol = ulp_tol(ref) + rope_shift(wq)
            self.note("q", (np.abs(q[:, hq] - ref) - tol + 1e-2).max())
        pg = tabs[task, pos // 16]
        for hk in kh:
            wk = self.W(l, OW.TID_QKV, range((nq + hk) * hd, (nq + hk + 1) * hd), d)
            wv = self.W(l, OW.TID_QKV, range((nq + nkv + hk) * hd, (nq + nkv + hk + 1) * hd), d)
            refk = bf16(rope((h @ wk.T)[:, None, :], pos, hd)[:, 0])
            refv = bf16(h @ wv.T)
            gk = bf(kv[pg, 0, hk, pos % 16])
            gv = bf(kv[pg, 1, hk, pos % 16])
            self.note("k_page", (np.abs(gk - refk) - ulp_tol(refk) - rope_shift(wk) + 1e-2).max())
            self.note("v_page", (np.abs(gv - refv) - ulp_tol(refv) - np.abs(dh @ wv.T) + 1e-2).max())
        # ---- attention on the GPU's q and pages (sampled rows, every head)
        for i in attn_rows:
            pages = tabs[task[i], :pos[i] // 16 + 1]
            kp = bf(kv[pages, 0]).transpose(0, 2, 1, 3)   # [page][slot][kv head][hd], this row's pages
            vp = bf(kv[pages, 1]).transpose(0, 2, 1, 3)
            ref = paged_attention(q[i], kp, vp, np.arange(len(pages)), pos[i] + 1)
            self.note("attn", (np.abs(o[i] - ref) - ulp_tol(ref) + 1e-2).max())
        # ---- O + residual (sampled output features)
        fo = np.sort(rng.choice(d, 384, replace=False))
        ref = x[:, fo] + o.reshape(n, nq * hd) @ self.W(l, OW.TID_O, fo, nq * hd).T
        self.note("x_after_o", np.abs(xm[:, fo] - ref).max() / np.sqrt(nq * hd / 512))
        # ---- gate/up + SwiGLU (sampled features: gate row f, up row ff + f); R-NORM shift
        # propagated to first order: |silu'(g) u dg| + |silu(g) du|
        ffs = np.sort(rng.choice(ff, 256, replace=False))
        h2 = bf16(rms(xm))
        dh2 = bf16(xm) / np.sqrt(np.mean(xm * xm, axis=-1, keepdims=True) + 1e-5) - h2
        wg, wu = self.W(l, OW.TID_GU, ffs, d), self.W(l, OW.TID_GU, ffs + ff, d)
        g, u = h2 @ wg.T, h2 @ wu.T
        ref = bf16(silu(g) * u)
        sg = 1.0 / (1.0 + np.exp(-g))
        dsilu = sg * (1.0 + g * (1.0 - sg))
        shift = np.abs(dsilu * u * (dh2 @ wg.T)) + np.abs(silu(g) * (dh2 @ wu.T))
        self.note("swiglu", (np.abs(act[:, ffs] - ref) - ulp_tol(ref) - 1.5 * shift + 1e-2).max())
        # ---- down + residual
        fd = np.sort(rng.choice(d, 384, replace=False))
        ref = xm[:, fd] + act @ self.W(l, OW.TID_D, fd, ff).T
        self.note("x_after_down", np.abs(xo[:, fd] - ref).max() / np.sqrt(ff / 512))


def run_fullsize(rt, shape, gemm_path=0, n_dec=64, n_tail=8, seed=31, mixed=True):
    """64 drone requests (1300-token private prompts, contexts >= 1300 after the first
    decode rounds) decoding, then n_tail requests whose prompts start with the registered
    1216-token drone prefix: the checked round has 64 decode rows + 8 x 84 prefill rows."""
    v = make_vocab(shape.vocab)
    plan = 40
    pages = n_dec * ((1300 + plan + 15) // 16 + 1) + n_tail * ((84 + plan + 15) // 16 + 1) + 76 + 16
    p = engine_params("b200-roofline", max_batch=n_dec + n_tail, max_tasks=2 * (n_dec + n_tail), max_ctx=1536,
                      n_pages=pages, max_seg_tokens=16)
    eng = rt.Engine(shape, p, v, seed=seed, flags=rt.RT_FLAG_CAPTURE_LAYERS, max_rows_per_forward=1024,
                    gemm_path=gemm_path)
    pfx = system_prefix(v, "drone", 1216, seed=seed)
    eng.register_prefix(pfx)
    for a in range(n_dec):
        tr = make_trace(1 + a % 5, v, seed=1000 + a, plan_len=plan)   # drone-normal plans, 1300-token prompt
        eng.submit(a, tr.prompt, 0, 100_000_000, -2.0, 1.0, 2 ** 31 - 1, script=tr.plan)
    # prefill rounds (84 k rows in 1024-row forward chunks), then decode until all 64 run
    for _ in range(200):
        info = eng.step()
        if info["n_running"] == n_dec and info["n_prefill_rows"] == 0:
            break
    assert info["n_running"] == n_dec and info["n_prefill_rows"] == 0, info
    checked = []

    def check_round(label):
        rows = eng.dump(rt.RT_DUMP_ROWS, np.int32).reshape(-1, 3)
        assert len(rows) <= 1024
        tabs = eng.dump(rt.RT_DUMP_PAGE_TABLES, np.int32).reshape(p.max_tasks, -1)
        rows_l = [(int(a), int(b)) for a, b, _ in rows]
        rng = np.random.default_rng(len(rows) + 7 * len(checked))
        pre = [i for i, (t, pp) in enumerate(rows_l) if pp < 1300]   # prompt rows (shared-prefix tails)
        attn_rows = sorted(set(int(i) for i in rng.choice(len(rows), min(24, len(rows)), replace=False))
                           | {0, len(rows) - 1} | set(pre[:3]) | set(pre[-3:]))
        ck = Checker(shape, seed)
        for l in range(shape.n_layers):
            ck.layer(eng, rt, l, rows_l, tabs, rng, attn_rows)
        checked.append((label, len(rows), ck.worst))
        return ck.worst

    w_dec = check_round("decode")
    if not mixed:
        eng.close()
        return w_dec, None, checked
    # the mixed round: n_tail prefix-sharing requests admitted next to the 64 running ones
    for a in range(n_tail):
        tr = make_trace(1 + a % 5, v, seed=5000 + a, prefix=pfx, plan_len=plan)
        eng.submit(n_dec + a, tr.prompt, 0, 100_000_000, -2.0, 1.0, 2 ** 31 - 1, script=tr.plan)
    info = eng.step()
    assert info["n_prefill_rows"] == n_tail * 84 and info["n_rows"] == n_dec + n_tail * 84, info
    w_mix = check_round("decode+prefill")
    eng.close()
    return w_dec, w_mix, checked


def assert_within(w):
    assert w["q"] < 1e-2, w
    assert w["k_page"] < 1e-2, w
    assert w["v_page"] < 1e-2, w
    assert w["attn"] < 1e-2, w
    assert w["swiglu"] < 1e-2, w
    assert w["x_after_o"] < 1e-3, w
    assert w["x_after_down"] < 1e-3, w


@pytest.mark.parametrize("gemm_path", [0, 1, 2, 3])
def test_llama8b_dims_every_fused_op_vs_oracle(rt, gemm_path):
    """8B layer dims (d 4096, 32 q / 8 kv heads, hd 128, ff 14336), 2 layers; the decode round
    runs the cluster split-K kernel at N = 64 (EPI_QKV / EPI_RESID / EPI_SWIGLU, folded RMSNorm),
    the mixed round's 736 rows the prefill kernels (gemm_path: the dispatch table, or forced
    one-tile-per-CTA / hybrid stream-K / CTA pairs) and the causal prefill attention."""
    s8 = MODEL_SHAPES["llama3-8b"]
    shape = ModelShape("8b-2l", 2, s8.d_model, s8.n_q_heads, s8.n_kv_heads, s8.head_dim, s8.d_ff, s8.vocab)
    w_dec, w_mix, checked = run_fullsize(rt, shape, gemm_path)
    print(checked)
    assert_within(w_dec)
    assert_within(w_mix)


def test_llama70b_dims_every_fused_op_vs_oracle(rt):
    """70B layer dims (d 8192, 64 q / 8 kv heads: G = 8, ff 28672), 2 layers, same rounds."""
    s7 = MODEL_SHAPES["llama3-70b"]
    shape = ModelShape("70b-2l", 2, s7.d_model, s7.n_q_heads, s7.n_kv_heads, s7.head_dim, s7.d_ff, s7.vocab)
    w_dec, w_mix, checked = run_fullsize(rt, shape, 0)
    print(checked)
    assert_within(w_dec)
    assert_within(w_mix)


@pytest.mark.parametrize("n_dec,gemm_path", [(256, 0), (200, 0), (64, 4), (128, 4)])
def test_llama8b_dims_decode_pair_splitk_vs_oracle(rt, n_dec, gemm_path):
    """The C3 decode round (256 rows; 200 = a ragged batch) runs QKV / O / down on the CTA-pair
    cluster split-K kernel (k_gemm_dec: QKV 24 pair-tiles x 3 splits, O / down 16 x 4) and
    gate/up on the persistent pair kernel; 64 / 128 rows force k_gemm_dec (gemm_path 4) at
    BN = 64 / 128.  Every fused op of both layers vs the oracle on the GPU's own inputs."""
    s8 = MODEL_SHAPES["llama3-8b"]
    shape = ModelShape("8b-2l", 2, s8.d_model, s8.n_q_heads, s8.n_kv_heads, s8.head_dim, s8.d_ff, s8.vocab)
    w_dec, _, checked = run_fullsize(rt, shape, gemm_path, n_dec=n_dec, n_tail=0, mixed=False)
    print(checked)
    assert_within(w_dec)


@pytest.mark.parametrize("n_dec,n_tail", [(64, 2), (32, 1)])
def test_llama8b_dims_mixed_fold_vs_oracle(rt, n_dec, n_tail):
    """Mixed rounds of <= 256 rows (decode rows + shared-prefix prompt tails, 232 / 116 rows):
    the QKV projection writes raw split-K partials, the decode attention runs the folded QKV
    epilogue of the decode rows and k_qkv_finish that of the prompt rows (q for the prefill
    attention, K/V appended); at > 128 rows O / down also write partials finished by the
    residual reduce.  Every fused op of both layers vs the oracle on the GPU's own inputs."""
    s8 = MODEL_SHAPES["llama3-8b"]
    shape = ModelShape("8b-2l", 2, s8.d_model, s8.n_q_heads, s8.n_kv_heads, s8.head_dim, s8.d_ff, s8.vocab)
    w_dec, w_mix, checked = run_fullsize(rt, shape, 0, n_dec=n_dec, n_tail=n_tail)
    print(checked)
    assert_within(w_dec)
    assert_within(w_mix)
