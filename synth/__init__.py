"""Seeded synthetic workloads shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no sharing, no PRG, no ring
GEMM): it only draws plaintext fixed-point inputs with numpy's seeded
generator and lists the paper's layer shapes.  Recipe: DESIGN.md §"Input
recipe".
"""
from __future__ import annotations

import numpy as np

MASTER_SEED = 210900984          # §8(d): master seed of every config
FRAC_BITS = 16                   # P:244 §7 "L = 16 by default"


def to_ring(v_int: np.ndarray) -> np.ndarray:
    """Two's-complement view of signed integers as ring elements (uint64)."""
    return np.ascontiguousarray(np.asarray(v_int, dtype=np.int64).view(np.uint64))


def uniform_fixed(shape, seed: int, bound: float = 8.0, frac_bits: int = FRAC_BITS) -> np.ndarray:
    """Integer fixed-point values U{-bound*2^f .. bound*2^f} as uint64 (configs C1/C2/C5)."""
    rng = np.random.default_rng(seed)
    lim = int(bound * (1 << frac_bits))
    return to_ring(rng.integers(-lim, lim + 1, size=shape, dtype=np.int64))


def gaussian_fixed(shape, seed: int, std: float, lo: float, hi: float, absval: bool = False,
                   frac_bits: int = FRAC_BITS) -> np.ndarray:
    """Clipped Gaussian values already on the 2^-f grid (configs C3/C4)."""
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(size=shape) * std
    if absval:
        v = np.abs(v)
    v = np.clip(v, lo, hi)
    return to_ring(np.rint(v * (1 << frac_bits)).astype(np.int64))


def uniform_ring(shape, seed: int) -> np.ndarray:
    """Full-range uniform ring elements (edge/stress cases)."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, 2**64 - 1, size=shape, dtype=np.uint64, endpoint=True)


# --- layer shapes (M, K, N, count), SURVEY.md §8(d) C3/C4 -----------------
RESNET50_B1 = [
    ("conv1", 12544, 147, 64, 1),
    ("l1.c1", 3136, 64, 64, 1), ("l1.c2", 3136, 576, 64, 3), ("l1.c3", 3136, 64, 256, 4),
    ("l1.c1b", 3136, 256, 64, 2),
    ("l2.c1", 3136, 256, 128, 1), ("l2.c2", 784, 1152, 128, 4), ("l2.c3", 784, 128, 512, 4),
    ("l2.ds", 784, 256, 512, 1), ("l2.c1b", 784, 512, 128, 3),
    ("l3.c1", 784, 512, 256, 1), ("l3.c2", 196, 2304, 256, 6), ("l3.c3", 196, 256, 1024, 6),
    ("l3.ds", 196, 512, 1024, 1), ("l3.c1b", 196, 1024, 256, 5),
    ("l4.c1", 196, 1024, 512, 1), ("l4.c2", 49, 4608, 512, 3), ("l4.c3", 49, 512, 2048, 3),
    ("l4.ds", 49, 1024, 2048, 1), ("l4.c1b", 49, 2048, 512, 2),
    ("fc", 1, 2048, 1000, 1),
]

VIT_B16 = [
    ("patch_embed", 196, 768, 768, 1),
    ("qkv", 197, 768, 2304, 12), ("proj", 197, 768, 768, 12),
    ("fc1", 197, 768, 3072, 12), ("fc2", 197, 3072, 768, 12),
    ("head", 1, 768, 1000, 1),
]

# ViT-B/16 with the attention matmuls (SURVEY §8(d) C4 "optional attention"): per
# block the 12 heads' Q @ K^T (197 x 64 x 197) and A @ V (197 x 197 x 64) as one
# batched private matmul each (6th field = batch).  Softmax is out of scope.
VIT_B16_ATTN = VIT_B16[:2] + [("qk^T", 197, 64, 197, 12, 12), ("attn@v", 197, 197, 64, 12, 12)] + VIT_B16[2:]

# ResNet-18 b1 im2col GEMMs (the model the paper benchmarks; SURVEY §8(d)
# C3 extra row): 21 GEMMs, sum MNK = 1.81 G.
RESNET18_B1 = [
    ("conv1", 12544, 147, 64, 1),
    ("l1.c", 3136, 576, 64, 4),
    ("l2.c1", 784, 576, 128, 1), ("l2.c", 784, 1152, 128, 3), ("l2.ds", 784, 64, 128, 1),
    ("l3.c1", 196, 1152, 256, 1), ("l3.c", 196, 2304, 256, 3), ("l3.ds", 196, 128, 256, 1),
    ("l4.c1", 49, 2304, 512, 1), ("l4.c", 49, 4608, 512, 3), ("l4.ds", 49, 256, 512, 1),
    ("fc", 1, 512, 1000, 1),
]

# Wav2Letter, 1 s of 16 kHz audio, batch 1 (SURVEY §8(d) optional row W,
# torchaudio padding assumed): sum MNK = 1.33 G.
WAV2LETTER_B1 = [
    ("conv1", 100, 250, 250, 1), ("conv2", 50, 12000, 250, 1), ("conv3-9", 50, 1750, 250, 7),
    ("conv10", 51, 8000, 2000, 1), ("conv11", 51, 2000, 2000, 1), ("conv12", 51, 2000, 29, 1),
]

# The same networks as true convolutions: (name, C, H, W, Cout,
# k, stride, pad, count), batch 1, torchvision ResNet v1.5 (stride in the 3x3 conv);
# the fc layer is a 1x1 convolution on a 1x1 map.  Same GEMM shapes as the lists above.
RESNET50_CONV_B1 = [
    ("conv1", 3, 224, 224, 64, 7, 2, 3, 1),
    ("l1.b1.c1", 64, 56, 56, 64, 1, 1, 0, 1), ("l1.c2", 64, 56, 56, 64, 3, 1, 1, 3),
    ("l1.c3", 64, 56, 56, 256, 1, 1, 0, 3), ("l1.ds", 64, 56, 56, 256, 1, 1, 0, 1),
    ("l1.c1", 256, 56, 56, 64, 1, 1, 0, 2),
    ("l2.b1.c1", 256, 56, 56, 128, 1, 1, 0, 1), ("l2.b1.c2", 128, 56, 56, 128, 3, 2, 1, 1),
    ("l2.c3", 128, 28, 28, 512, 1, 1, 0, 4), ("l2.ds", 256, 56, 56, 512, 1, 2, 0, 1),
    ("l2.c1", 512, 28, 28, 128, 1, 1, 0, 3), ("l2.c2", 128, 28, 28, 128, 3, 1, 1, 3),
    ("l3.b1.c1", 512, 28, 28, 256, 1, 1, 0, 1), ("l3.b1.c2", 256, 28, 28, 256, 3, 2, 1, 1),
    ("l3.c3", 256, 14, 14, 1024, 1, 1, 0, 6), ("l3.ds", 512, 28, 28, 1024, 1, 2, 0, 1),
    ("l3.c1", 1024, 14, 14, 256, 1, 1, 0, 5), ("l3.c2", 256, 14, 14, 256, 3, 1, 1, 5),
    ("l4.b1.c1", 1024, 14, 14, 512, 1, 1, 0, 1), ("l4.b1.c2", 512, 14, 14, 512, 3, 2, 1, 1),
    ("l4.c3", 512, 7, 7, 2048, 1, 1, 0, 3), ("l4.ds", 1024, 14, 14, 2048, 1, 2, 0, 1),
    ("l4.c1", 2048, 7, 7, 512, 1, 1, 0, 2), ("l4.c2", 512, 7, 7, 512, 3, 1, 1, 2),
    ("fc", 2048, 1, 1, 1000, 1, 1, 0, 1),
]
RESNET18_CONV_B1 = [
    ("conv1", 3, 224, 224, 64, 7, 2, 3, 1),
    ("l1.c", 64, 56, 56, 64, 3, 1, 1, 4),
    ("l2.b1.c1", 64, 56, 56, 128, 3, 2, 1, 1), ("l2.c", 128, 28, 28, 128, 3, 1, 1, 3),
    ("l2.ds", 64, 56, 56, 128, 1, 2, 0, 1),
    ("l3.b1.c1", 128, 28, 28, 256, 3, 2, 1, 1), ("l3.c", 256, 14, 14, 256, 3, 1, 1, 3),
    ("l3.ds", 128, 28, 28, 256, 1, 2, 0, 1),
    ("l4.b1.c1", 256, 14, 14, 512, 3, 2, 1, 1), ("l4.c", 512, 7, 7, 512, 3, 1, 1, 3),
    ("l4.ds", 256, 14, 14, 512, 1, 2, 0, 1),
    ("fc", 512, 1, 1, 1000, 1, 1, 0, 1),
]
CONV_MODELS = {"resnet50": RESNET50_CONV_B1, "resnet18": RESNET18_CONV_B1}

# Wav2Letter as true 1-D convolutions: torchaudio's
# waveform model, 1 s of 16 kHz audio, 29 classes: (name, C, L, Cout, k, stride, pad,
# count).  Same im2col GEMM shapes as WAV2LETTER_B1 (M = B * L_out, K = C * k, N = Cout).
WAV2LETTER_CONV1D = [
    ("conv1", 1, 16000, 250, 250, 160, 45, 1),
    ("conv2", 250, 100, 250, 48, 2, 23, 1),
    ("conv3-9", 250, 50, 250, 7, 1, 3, 7),
    ("conv10", 250, 50, 2000, 32, 1, 16, 1),
    ("conv11", 2000, 51, 2000, 1, 1, 0, 1),
    ("conv12", 2000, 51, 29, 1, 1, 0, 1),
]

# Text classification: the embedding applied as a
# dense matmul of 32 one-hot tokens x vocabulary 519,820 x embedding 32 — a wide
# reduction (K >> 16512, the per-unit exactness bound) at tiny M and N.
TEXT_EMBED = [("embed", 32, 519820, 32, 1)]

MODELS = {"resnet50": RESNET50_B1, "vit": VIT_B16, "resnet18": RESNET18_B1, "wav2letter": WAV2LETTER_B1,
          "text": TEXT_EMBED, "vit_attn": VIT_B16_ATTN}

CONFIGS = {
    "C1": dict(M=64, K=64, N=64, P=2, seed=1001),
    "C2": dict(M=4096, K=4096, N=4096, P=2, seed=1002),
    "C5": dict(M=8192, K=8192, N=8192, P=8, seed=1005),
}
