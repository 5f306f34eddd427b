"""Counter-based random init (oracle side; test infrastructure only).

SURVEY AMB-15 (the build's reading of BASELINE.json "random-init"):
    u = splitmix64(seed ^ (tensor_id << 40) ^ idx)
    w = bf16_rne( ((u >> 40) * 2^-24 - 0.5) * c ),  c = fp32(2*sqrt(3)*sigma)
i.e. uniform with standard deviation sigma (HF default 0.02).  Everything
before the final fp32 multiply is exact; the multiply and the bf16 rounding are
single RNE steps, so the CUDA side can reproduce the weights bit for bit with
an independent implementation.

tensor_id: embedding 0, lm_head 1, layer l: 16 + 8 l + {0: W_qkv, 1: W_o,
2: W_gate_up, 3: W_down}.  idx = row * in_features + col of the logical
[out, in] matrix.  W_qkv rows = [q heads | k heads | v heads]; W_gate_up rows
= [gate | up].
"""
import math
import numpy as np

from .bf16 import bf16_bits, bits_to_f32

M64 = (1 << 64) - 1
TID_EMB, TID_LM = 0, 1
TID_QKV, TID_O, TID_GU, TID_D = 0, 1, 2, 3


def layer_tid(layer: int, j: int) -> int:
    return 16 + 8 * layer + j


def splitmix64_int(x: int) -> int:
    """Reference scalar splitmix64 (Steele/Lea/Flood), pure Python ints."""
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def scale_const(sigma: float) -> np.float32:
    return np.float32(2.0 * math.sqrt(3.0) * sigma)


def weight_values(seed: int, tensor_id: int, idx, sigma: float = 0.02) -> np.ndarray:
    """fp32 array holding the bf16 weight values at flat indices ``idx``."""
    idx = np.asarray(idx, dtype=np.uint64)
    key = np.uint64(seed & M64) ^ (np.uint64(tensor_id) << np.uint64(40))
    u = splitmix64(key ^ idx)
    r = (u >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24) - np.float32(0.5)
    w = (r * scale_const(sigma)).astype(np.float32)
    return bits_to_f32(bf16_bits(w))


def matrix(seed: int, tensor_id: int, rows, n_in: int, sigma: float = 0.02) -> np.ndarray:
    """Rows ``rows`` (iterable or range) of a logical [out, n_in] weight, float64."""
    rows = np.asarray(list(rows) if not isinstance(rows, np.ndarray) else rows, dtype=np.uint64)
    idx = rows[:, None] * np.uint64(n_in) + np.arange(n_in, dtype=np.uint64)[None, :]
    return weight_values(seed, tensor_id, idx, sigma).astype(np.float64)
