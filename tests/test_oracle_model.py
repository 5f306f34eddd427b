"""Pins for oracle c1 (model), the bf16 materialisation (P12), the counter-based
init (AMB-15) and paged attention (P6).  Library routines and closed forms,
never the oracle's own formulas retyped."""
import numpy as np
import pytest
import torch

from oracle import weights as W
from oracle.bf16 import bf16, bf16_bits
from oracle.model import OracleModel, dense_attention, paged_attention, rope
from synth import MODEL_SHAPES
from synth.configs import ModelShape


def test_p12_bf16_rne_matches_torch():
    rng = np.random.default_rng(0)
    u = rng.integers(0, 2 ** 32, size=2_000_000, dtype=np.uint64).astype(np.uint32)
    f = u.view(np.float32)
    f = f[np.isfinite(f)]
    mine = bf16_bits(f)
    ref = torch.from_numpy(f.copy()).bfloat16().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(mine, ref)
    # ties to even: 1 + 2^-8 is a tie between 1 and 1 + 2^-7 -> rounds to even mantissa (1.0)
    assert bf16(np.float32(1.0 + 2 ** -8)) == 1.0
    assert bf16(np.float32(1.0 + 3 * 2 ** -8)) == 1.0 + 2 ** -6


def test_splitmix64_known_vectors():
    # SplitMix64 (Steele, Lea, Flood 2014) seeded with 0: published first outputs
    state = 0
    outs = []
    for _ in range(3):
        outs.append(W.splitmix64_int(state))
        state = (state + 0x9E3779B97F4A7C15) & W.M64
    assert outs == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    x = np.array([0, 0x9E3779B97F4A7C15, 2 * 0x9E3779B97F4A7C15 & W.M64], dtype=np.uint64)
    assert [int(v) for v in W.splitmix64(x)] == outs


def test_weight_init_distribution_and_exactness():
    sigma = 0.02
    w = W.weight_values(1234, 7, np.arange(1 << 20, dtype=np.uint64), sigma)
    half = np.sqrt(3.0) * sigma
    assert w.min() >= -half * (1 + 2 ** -8) and w.max() <= half * (1 + 2 ** -8)
    assert abs(w.mean()) < 3 * sigma / np.sqrt(len(w)) * 3
    assert w.std() == pytest.approx(sigma, rel=5e-3)
    # bf16-representable, deterministic, tensor ids decorrelated
    assert np.array_equal(bf16(w).astype(np.float32), w)
    assert np.array_equal(w, W.weight_values(1234, 7, np.arange(1 << 20, dtype=np.uint64), sigma))
    w2 = W.weight_values(1234, 8, np.arange(1 << 20, dtype=np.uint64), sigma)
    assert abs(np.corrcoef(w, w2)[0, 1]) < 0.01
    # closed form for one element, computed independently with Python ints/floats
    idx, seed, tid = 12345, 1234, 7
    u = W.splitmix64_int(seed ^ (tid << 40) ^ idx)
    r = np.float32((u >> 40) / 2 ** 24 - 0.5)
    expect = torch.tensor(float(np.float32(r * np.float32(2 * 3 ** 0.5 * sigma)))).bfloat16().item()
    assert float(W.weight_values(seed, tid, [idx], sigma)[0]) == expect


def test_rope_closed_form():
    hd = 32
    rng = np.random.default_rng(1)
    q = rng.standard_normal((1, 2, hd))
    k = rng.standard_normal((1, 2, hd))
    for p1, p2 in [(3, 10), (100, 107), (0, 7)]:
        a = (rope(q, [p1], hd) * rope(k, [p2], hd)).sum()
        b = (rope(q, [p1 + 50], hd) * rope(k, [p2 + 50], hd)).sum()
        assert a == pytest.approx(b, rel=1e-10)          # relative-position property
    assert np.allclose(np.linalg.norm(rope(q, [77], hd), axis=-1), np.linalg.norm(q, axis=-1))
    assert np.allclose(rope(q, [0], hd), q)


def test_p6_paged_attention_vs_sdpa_and_permutation():
    rng = np.random.default_rng(2)
    nq, nkv, hd, P = 8, 2, 64, 16
    T = 53
    n_pages = 10
    kp = rng.standard_normal((n_pages, P, nkv, hd))
    vp = rng.standard_normal((n_pages, P, nkv, hd))
    table = [7, 2, 9, 0]
    q = rng.standard_normal((nq, hd))
    o = paged_attention(q, kp, vp, table, T, P)
    pos = np.arange(T)
    K = kp[np.array(table)[pos // P], pos % P]
    V = vp[np.array(table)[pos // P], pos % P]
    G = nq // nkv
    qt = torch.from_numpy(q).view(1, nq, 1, hd)
    Kt = torch.from_numpy(np.repeat(K, G, axis=1)).permute(1, 0, 2).unsqueeze(0)
    Vt = torch.from_numpy(np.repeat(V, G, axis=1)).permute(1, 0, 2).unsqueeze(0)
    ref = torch.nn.functional.scaled_dot_product_attention(qt, Kt, Vt).view(nq, hd).numpy()
    assert np.allclose(o, ref, atol=1e-12, rtol=0)
    # permuting physical page ids does not change the result
    perm = rng.permutation(n_pages)
    inv = np.argsort(perm)
    o2 = paged_attention(q, kp[inv], vp[inv], [perm[i] for i in table], T, P)
    assert np.allclose(o, o2, atol=1e-14)


def _hf_llama(shape, om):
    from transformers import LlamaConfig, LlamaForCausalLM
    cfg = LlamaConfig(vocab_size=shape.vocab, hidden_size=shape.d_model, intermediate_size=shape.d_ff,
                      num_hidden_layers=shape.n_layers, num_attention_heads=shape.n_q_heads,
                      num_key_value_heads=shape.n_kv_heads, head_dim=shape.head_dim,
                      rms_norm_eps=1e-5, rope_theta=500000.0, tie_word_embeddings=False,
                      attention_bias=False, mlp_bias=False, max_position_embeddings=4096)
    m = LlamaForCausalLM(cfg).double().eval()
    s = shape
    nq, nkv, hd = s.n_q_heads, s.n_kv_heads, s.head_dim
    with torch.no_grad():
        m.model.embed_tokens.weight.copy_(torch.from_numpy(om.emb_rows(range(s.vocab))))
        m.lm_head.weight.copy_(torch.from_numpy(om.lm()))
        for l, layer in enumerate(m.model.layers):
            w = om.layer(l)
            qkv = torch.from_numpy(w["qkv"])
            layer.self_attn.q_proj.weight.copy_(qkv[:nq * hd])
            layer.self_attn.k_proj.weight.copy_(qkv[nq * hd:(nq + nkv) * hd])
            layer.self_attn.v_proj.weight.copy_(qkv[(nq + nkv) * hd:])
            layer.self_attn.o_proj.weight.copy_(torch.from_numpy(w["o"]))
            gu = torch.from_numpy(w["gu"])
            layer.mlp.gate_proj.weight.copy_(gu[:s.d_ff])
            layer.mlp.up_proj.weight.copy_(gu[s.d_ff:])
            layer.mlp.down_proj.weight.copy_(torch.from_numpy(w["d"]))
    return m


@pytest.mark.parametrize("shape", [MODEL_SHAPES["tiny"], ModelShape("g2", 2, 64, 4, 2, 16, 96, 300)])
def test_p7_model_equals_transformers(shape):
    om = OracleModel(shape, seed=5, bf16_points=False)
    hf = _hf_llama(shape, om)
    rng = np.random.default_rng(3)
    toks = rng.integers(0, shape.vocab, size=12)
    with torch.no_grad():
        ref = hf(torch.from_numpy(toks).view(1, -1)).logits[0].numpy()
    # prefill rows 0..7 in one forward, then decode rows 8..11 one at a time (KV reuse)
    rows = [(0, i, int(toks[i])) for i in range(8)]
    h = om.forward(rows)
    got = [om.logits(h)]
    for i in range(8, 12):
        got.append(om.logits(om.forward([(0, i, int(toks[i]))])))
    got = np.concatenate(got)
    # HF keeps inv_freq / cos / sin in fp32 even in a float64 model -> ~1e-8 differences
    assert np.allclose(got, ref, atol=1e-6, rtol=0)


def test_bf16_points_drift_small_tiny():
    # Appendix A of SURVEY: bf16 points move tiny-model logits by ~1e-3
    shape = MODEL_SHAPES["tiny"]
    a = OracleModel(shape, seed=5, bf16_points=False)
    b = OracleModel(shape, seed=5, bf16_points=True)
    rows = [(0, i, t) for i, t in enumerate([5, 77, 300, 12, 9])]
    la = a.logits(a.forward(rows))
    lb = b.logits(b.forward(rows))
    assert np.max(np.abs(la - lb)) < 2e-2


def test_dense_attention_softmax_rows():
    rng = np.random.default_rng(4)
    q = rng.standard_normal((4, 16))
    K = rng.standard_normal((1, 1, 16)).repeat(9, axis=0)   # identical keys -> uniform weights
    V = rng.standard_normal((9, 1, 16))
    o = dense_attention(q, K, V)
    assert np.allclose(o, V[:, 0, :].mean(axis=0)[None, :].repeat(4, 0), atol=1e-12)
