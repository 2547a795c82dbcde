"""Seeded synthetic inputs for BASELINE.json configs 0-4.

The paper's datasets (ViT/MPNet features of MNIST, CIFAR-10, ...) are not
available offline; these generators reproduce the shapes, sizes and value
distributions BASELINE.json names.  One module fixes the draw order so the
GPU path, the CPU oracle and the float64 twin see identical inputs.
"""

from __future__ import annotations

import numpy as np

CLASSES = 10
FEATURES = 768
BATCH = 128


def _rownorm(x: np.ndarray) -> np.ndarray:
    return x / np.linalg.norm(x, axis=1, keepdims=True)


def softmax_rows(z: np.ndarray) -> np.ndarray:
    e = np.exp(z - z.max(axis=1, keepdims=True))
    return e / e.sum(axis=1, keepdims=True)


def config0():
    """DiagABT plumbing check: A (64x64), B (16x64), U[-1,1], seed 0 (A first)."""
    rng = np.random.default_rng(0)
    A = rng.uniform(-1.0, 1.0, size=(64, 64))
    B = rng.uniform(-1.0, 1.0, size=(16, 64))
    return A, B


def config1():
    """X (128x768) L2-normalised Gaussian rows, W (10x768) ~ N(0, 0.01^2), seed 1."""
    rng = np.random.default_rng(1)
    X = _rownorm(rng.standard_normal((BATCH, FEATURES)))
    W = 0.01 * rng.standard_normal((CLASSES, FEATURES))
    return X, W


def config2():
    """(P - Y) (128x10): softmax of N(0,1) logits minus one-hot labels, seed 2."""
    rng = np.random.default_rng(2)
    P = softmax_rows(rng.standard_normal((BATCH, CLASSES)))
    labels = rng.integers(0, CLASSES, size=BATCH)
    Y = np.zeros((BATCH, CLASSES))
    Y[np.arange(BATCH), labels] = 1.0
    X, _ = config1()
    return P - Y, X


def config3():
    """Softmax input: 128x10 logits ~ U[-128, 128], seed 3."""
    rng = np.random.default_rng(3)
    return rng.uniform(-128.0, 128.0, size=(BATCH, CLASSES))


def config4(rows: int = 1024):
    """10-class Gaussian mixture, 1024x768, class means N(0,1)/sqrt(768),
    within-class sigma 0.5, rows L2-normalised, seed 4; labels U{0..9}."""
    rng = np.random.default_rng(4)
    means = rng.standard_normal((CLASSES, FEATURES)) / np.sqrt(FEATURES)
    labels = rng.integers(0, CLASSES, size=rows)
    X = _rownorm(means[labels] + 0.5 * rng.standard_normal((rows, FEATURES)))
    return X, labels


LEARNING_RATE = 0.3  # training.py:269 default; BASELINE.json leaves lr unspecified
INIT_SEED = 4
