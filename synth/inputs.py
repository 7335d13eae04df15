"""Seeded input generators (SURVEY §8(d) seeds: data 2110, weights 13638,
keygen Philox 1, encryption Philox 2).

Readings: "N(0, s)" in BASELINE.json is a standard deviation (Z11);
biases follow the weights' law.  Fashion-MNIST and the agri-food data are absent:
uniform-uint8 28x28 images and standardised N(0,1) features stand in for their
shape and range.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

DATA_SEED = 2110
WEIGHT_SEED = 13638
KEY_SEED = 1
ENC_SEED = 2
RESIDUE_SEED = 3


@dataclass
class C0Inputs:
    X: np.ndarray      # (64, 16) in [0, 1)
    W: np.ndarray      # (4, 16)
    b: np.ndarray      # (4,)


def c0_inputs(seed_data: int = DATA_SEED, seed_w: int = WEIGHT_SEED, samples: int = 64) -> C0Inputs:
    rd = np.random.default_rng(seed_data)
    rw = np.random.default_rng(seed_w)
    X = rd.random((samples, 16))
    W = rw.normal(0.0, 0.25, (4, 16))
    b = rw.normal(0.0, 0.25, 4)
    return C0Inputs(X, W, b)


@dataclass
class C1Inputs:
    images: np.ndarray  # (B, 28, 28) float64 in [0, 1]
    K: np.ndarray       # (5, 4, 4)
    kb: np.ndarray      # (5,)
    W: np.ndarray       # (10, 245)
    b: np.ndarray       # (10,)


def c1_weights(seed_w: int = WEIGHT_SEED):
    rw = np.random.default_rng(seed_w)
    K = rw.normal(0.0, 0.1, (5, 4, 4))
    kb = rw.normal(0.0, 0.1, 5)
    W = rw.normal(0.0, 0.1, (10, 245))
    b = rw.normal(0.0, 0.1, 10)
    return K, kb, W, b


def c1_images(batch: int = 8192, seed_data: int = DATA_SEED) -> np.ndarray:
    rd = np.random.default_rng(seed_data)
    return rd.integers(0, 256, (batch, 28, 28)).astype(np.float64) / 255.0


def c1_inputs(batch: int = 8192, seed_data: int = DATA_SEED, seed_w: int = WEIGHT_SEED) -> C1Inputs:
    K, kb, W, b = c1_weights(seed_w)
    return C1Inputs(c1_images(batch, seed_data), K, kb, W, b)


def c1_slots(images: np.ndarray) -> np.ndarray:
    """Batch-in-slots packing: one ciphertext per pixel, slot s = image s -> (784, B)."""
    B = images.shape[0]
    return np.ascontiguousarray(images.reshape(B, 784).T)


@dataclass
class C3Inputs:
    X: np.ndarray      # (16384, 32) standardised
    W1: np.ndarray     # (64, 32)
    b1: np.ndarray
    W2: np.ndarray     # (1, 64)
    b2: np.ndarray


def c3_inputs(samples: int = 16384, seed_data: int = DATA_SEED, seed_w: int = WEIGHT_SEED) -> C3Inputs:
    rd = np.random.default_rng(seed_data)
    X = rd.normal(0.0, 1.0, (samples, 32))
    X = (X - X.mean(axis=0)) / X.std(axis=0)
    rw = np.random.default_rng(seed_w)
    W1 = rw.normal(0.0, 0.1, (64, 32))
    b1 = rw.normal(0.0, 0.1, 64)
    W2 = rw.normal(0.0, 0.1, (1, 64))
    b2 = rw.normal(0.0, 0.1, 1)
    return C3Inputs(X, W1, b1, W2, b2)


def random_residues(shape, moduli_per_row, seed: int = RESIDUE_SEED) -> np.ndarray:
    """Uniform residues: row r of the flattened [..., N] array is uniform in [0, moduli_per_row[r])."""
    rng = np.random.default_rng(seed)
    out = np.empty(shape, dtype=np.uint64)
    flat = out.reshape(-1, shape[-1])
    for r in range(flat.shape[0]):
        flat[r] = rng.integers(0, int(moduli_per_row[r]), shape[-1], dtype=np.uint64)
    return out


def random_slots(count: int, n_slots: int, seed: int = DATA_SEED, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, (count, n_slots))
