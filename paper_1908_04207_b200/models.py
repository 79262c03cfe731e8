"""Hyperplane-regression workload on the GPU (models.py:35-84 of the reference).

Not the hot path -- it produces the gradients the path consumes (BASELINE
config 1).  The dataset, the initial weights and the per-(rank, step)
minibatch indices are drawn with the reference's numpy generators, so a GPU run
sees exactly the reference's data; the model arithmetic runs in torch.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


@dataclass
class HyperplaneDataset:
    a: np.ndarray
    x_train: torch.Tensor
    y_train: torch.Tensor
    x_val: torch.Tensor
    y_val: torch.Tensor
    sigma: float
    seed: int

    @property
    def n_train(self) -> int:
        return self.x_train.shape[0]


def gen_dataset(dim: int = 64, n: int = 4096, sigma: float = 0.1, seed: int = 0,
                device=None, dtype=torch.float32) -> HyperplaneDataset:
    """models.py:35-44 (same generator calls, so the same samples)."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal(dim)
    x = rng.uniform(-1.0, 1.0, size=(n, dim))
    y = x @ a + sigma * rng.standard_normal(n)
    n_train = int(0.8 * n)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device

    def t(v):
        return torch.as_tensor(v, dtype=dtype, device=dev)

    return HyperplaneDataset(a=a, x_train=t(x[:n_train]), y_train=t(y[:n_train]),
                             x_val=t(x[n_train:]), y_val=t(y[n_train:]), sigma=sigma, seed=seed)


def init_weights(dim: int, seed: int = 0, scale: float = 0.01) -> np.ndarray:
    """models.py:53-56"""
    rng = np.random.default_rng(seed)
    return scale * rng.standard_normal(dim)


def loss_and_grad(w: torch.Tensor, x: torch.Tensor, y: torch.Tensor):
    """models.py:62-71: loss = (1/b) sum (w.x - y)^2, grad = (2/b) x^T (xw - y).
    Returns (loss tensor, grad tensor); both stay on the device."""
    r = x @ w - y
    b = x.shape[0]
    loss = (r @ r) / b
    grad = (2.0 / b) * (x.T @ r)
    return loss, grad


def mse(w: torch.Tensor, x: torch.Tensor, y: torch.Tensor) -> float:
    r = x @ w - y
    return float((r @ r) / x.shape[0])


def batch_indices(n_train: int, seed: int, rank: int, step: int, batch: int) -> np.ndarray:
    """models.py:79-84: the deterministic per-(rank, step) minibatch."""
    rng = np.random.default_rng([seed, rank, step])
    return rng.integers(0, n_train, size=batch)


def sample_batch(ds: HyperplaneDataset, seed: int, rank: int, step: int, batch: int):
    idx = torch.as_tensor(batch_indices(ds.n_train, seed, rank, step, batch),
                          device=ds.x_train.device)
    return ds.x_train[idx], ds.y_train[idx]
