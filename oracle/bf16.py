"""bf16 round-to-nearest-even materialisation (oracle, test infrastructure only).

SURVEY P12: numpy RNE on the uint32 view
    ((u + 0x7FFF + ((u >> 16) & 1)) >> 16)
equals torch.Tensor.bfloat16() bit-for-bit (pinned in tests/test_oracle_model.py).
"""
import numpy as np


def bf16_bits(x) -> np.ndarray:
    """float -> uint16 bf16 bit patterns (RNE from the fp32 value)."""
    f = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) & 0xFFFF
    nan = np.isnan(f)
    r = np.where(nan, (u >> 16) | 0x40, r)
    return r.astype(np.uint16)


def bits_to_f32(b) -> np.ndarray:
    b = np.ascontiguousarray(np.asarray(b, dtype=np.uint16))
    return (b.astype(np.uint32) << 16).view(np.float32)


def bf16(x) -> np.ndarray:
    """Round to the nearest bf16 value, returned as float64 (exactly representable)."""
    return bits_to_f32(bf16_bits(x)).astype(np.float64)
