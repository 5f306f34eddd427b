"""Llama-shaped decoder, decode/prefill rows (oracle c1, test infrastructure only).

SURVEY §8(c) c1 (the paper only names "Llama3-8B-float16"; the
decode-with-KV-cache model is BASELINE.json's "fp32 transformer decode with a
KV cache", "bf16 inputs, fp32 accumulate"):

  x = emb[tok]
  per layer:  h = rms(x);  q,k,v = h W_qkv^T;  RoPE rotate-half (pairs i, i+hd/2,
              theta = 500000, position = absolute index);  store bf16 k, v;
              o = softmax(q K^T / sqrt(hd)) V   (GQA: q head h -> kv head h // G)
              x += o W_o^T;  h = rms(x);  x += (silu(h W_g^T) * (h W_u^T)) W_d^T
  final:      h = rms(x);  logits = h W_lm^T;  token = argmax (lowest index on ties)
  rms(x) = x * rsqrt(mean(x^2) + 1e-5)   (gamma = 1)

Accumulation is fp64 here; bf16 RNE is applied at the materialisation points
SURVEY c1 fixes when ``bf16_points`` is True: GEMM inputs (h = rms(x), o, the
SwiGLU product), q after RoPE, stored K and V.  The residual stream x is not
rounded.  With ``bf16_points=False`` this is the plain model definition
(pinned against transformers.LlamaForCausalLM).

The CUDA path folds RMSNorm into the consuming projection: it rounds x (not
rms(x)) to bf16 and scales each output row by rsqrt(mean(x^2) + eps) in fp32
in the epilogue — the same algebra with the rounding point moved.  The oracle
keeps the definition above; reading R-NORM bounds the difference
(per-op tolerances of tests/test_gpu_fullsize.py).
"""
import numpy as np

from . import weights as W
from .bf16 import bf16

ROPE_THETA = 500000.0
RMS_EPS = 1e-5


def rms(x):
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + RMS_EPS)


def silu(g):
    return g / (1.0 + np.exp(-g))


def rope(x, pos, hd):
    """x: [n, heads, hd]; pos: [n] absolute positions. Rotate-half."""
    half = hd // 2
    inv = np.power(ROPE_THETA, -np.arange(half, dtype=np.float64) * 2.0 / hd)
    ang = np.asarray(pos, dtype=np.float64)[:, None] * inv[None, :]
    c = np.cos(ang)[:, None, :]
    s = np.sin(ang)[:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def dense_attention(q, K, V):
    """q: [nq, hd]; K, V: [T, nkv, hd] -> o [nq, hd]; softmax(q K^T / sqrt(hd)) V."""
    nq, hd = q.shape
    nkv = K.shape[1]
    G = nq // nkv
    o = np.empty((nq, hd), dtype=np.float64)
    for h in range(nq):
        kh = h // G
        s = K[:, kh, :] @ q[h] / np.sqrt(hd)
        s = s - s.max()
        p = np.exp(s)
        p = p / p.sum()
        o[h] = p @ V[:, kh, :]
    return o


def paged_attention(q, k_pages, v_pages, page_table, seq_len, page_tokens=16):
    """Attention over a page table (c2: paging is layout only).

    k_pages / v_pages: [n_pages, page_tokens, nkv, hd] logical page contents.
    Position p lives in page page_table[p // page_tokens], slot p % page_tokens.
    """
    pos = np.arange(seq_len)
    pages = np.asarray(page_table)[pos // page_tokens]
    K = k_pages[pages, pos % page_tokens]
    V = v_pages[pages, pos % page_tokens]
    return dense_attention(np.asarray(q, dtype=np.float64), K.astype(np.float64), V.astype(np.float64))


class OracleModel:
    """Random-init Llama decoder regenerated from the counter-based init (AMB-15)."""

    def __init__(self, shape, seed: int, sigma: float = 0.02, bf16_points: bool = True,
                 max_ctx: int = 4096):
        self.s = shape
        self.seed = seed
        self.sigma = sigma
        self.bf = bf16_points
        self.max_ctx = max_ctx
        self._layers = {}
        self._emb = None
        self._lm = None
        self.cache = {}  # req_id -> (K [L, max_ctx, nkv, hd], V)

    # ---- weights -------------------------------------------------------
    def _r(self, x):
        return bf16(x) if self.bf else x

    def emb_rows(self, toks):
        return W.matrix(self.seed, W.TID_EMB, np.asarray(toks, dtype=np.uint64), self.s.d_model, self.sigma)

    def lm(self):
        if self._lm is None:
            self._lm = W.matrix(self.seed, W.TID_LM, range(self.s.vocab), self.s.d_model, self.sigma)
        return self._lm

    def layer(self, l):
        if l not in self._layers:
            s = self.s
            d, hd = s.d_model, s.head_dim
            self._layers[l] = dict(
                qkv=W.matrix(self.seed, W.layer_tid(l, W.TID_QKV), range(s.qkv_dim), d, self.sigma),
                o=W.matrix(self.seed, W.layer_tid(l, W.TID_O), range(d), s.n_q_heads * hd, self.sigma),
                gu=W.matrix(self.seed, W.layer_tid(l, W.TID_GU), range(2 * s.d_ff), d, self.sigma),
                d=W.matrix(self.seed, W.layer_tid(l, W.TID_D), range(d), s.d_ff, self.sigma),
            )
        return self._layers[l]

    # ---- KV cache (logical, contiguous per request) ---------------------
    def _kv(self, rid):
        if rid not in self.cache:
            s = self.s
            shp = (s.n_layers, self.max_ctx, s.n_kv_heads, s.head_dim)
            self.cache[rid] = (np.zeros(shp), np.zeros(shp))
        return self.cache[rid]

    def drop(self, rid):
        self.cache.pop(rid, None)

    def share_prefix(self, src, dst, n):
        """Request dst starts with the n positions of registered prefix src: the keys and
        values of a position depend only on the tokens up to it, so they are the prefix's."""
        K, V = self._kv(src)
        K2, V2 = self._kv(dst)
        K2[:, :n] = K[:, :n]
        V2[:, :n] = V[:, :n]

    # ---- forward over a set of rows --------------------------------------
    def forward(self, rows, capture=None):
        """rows: list of (req_id, pos, token).  Returns final-normed hidden (bf16
        points applied) for every row, shape [n, d].  ``capture`` (optional dict)
        receives per-layer q / o for per-op parity."""
        s = self.s
        nq, nkv, hd = s.n_q_heads, s.n_kv_heads, s.head_dim
        toks = [r[2] for r in rows]
        pos = np.array([r[1] for r in rows])
        x = self.emb_rows(toks)
        n = len(rows)
        for l in range(s.n_layers):
            w = self.layer(l)
            h = self._r(rms(x))
            qkv = h @ w["qkv"].T
            q = qkv[:, :nq * hd].reshape(n, nq, hd)
            k = qkv[:, nq * hd:(nq + nkv) * hd].reshape(n, nkv, hd)
            v = qkv[:, (nq + nkv) * hd:].reshape(n, nkv, hd)
            q = self._r(rope(q, pos, hd))
            k = self._r(rope(k, pos, hd))
            v = self._r(v)
            for i, (rid, p, _) in enumerate(rows):
                K, V = self._kv(rid)
                K[l, p] = k[i]
                V[l, p] = v[i]
            o = np.empty((n, nq, hd))
            for i, (rid, p, _) in enumerate(rows):
                K, V = self._kv(rid)
                o[i] = dense_attention(q[i], K[l, :p + 1], V[l, :p + 1])
            if capture is not None:
                capture.setdefault("q", []).append(q.copy())
                capture.setdefault("o", []).append(o.copy())
            x = x + self._r(o.reshape(n, nq * hd)) @ w["o"].T
            h = self._r(rms(x))
            gu = h @ w["gu"].T
            a = self._r(silu(gu[:, :s.d_ff]) * gu[:, s.d_ff:])
            x = x + a @ w["d"].T
        return self._r(rms(x))

    def logits(self, hidden):
        return hidden @ self.lm().T


def argmax_lowest(v) -> int:
    """numpy argmax returns the first maximum, i.e. the lowest index (c3)."""
    return int(np.argmax(v))
