"""BASELINE config 4 workload: an LSTM on UCF101-shaped synthetic sequences.

The paper's third experiment trains a single-layer
LSTM video classifier on UCF101 frame features; per-sample sequence lengths
range over 29-1,776 frames (mean 187, sd 97), so ranks that draw long videos
straggle -- imbalance that is inherent, not injected.  The reference package
has no such workload (SPEC.md:16 puts it out of scope); here it exists only to
drive the eager-SGD path with a real model:

* weights and gradients live in flat fp32 buffers: the parameters are views
  into `TrainState.w`, and the gradients are views into the collective's
  registered gradient bucket, so backward writes the gradient where the
  reduction reads it (zero-copy offer) and the update writes the weights the
  next forward uses;
* per-rank minibatches of `batch` sequences with UCF101-shaped lengths, padded
  to the batch maximum (the straggler effect), random 2048-d features and
  labels over 101 classes (synthetic data; no network access for the dataset).
"""

from __future__ import annotations

import numpy as np
import torch

FEATURES = 2048      # InceptionV3 pool features per frame
HIDDEN = 2048        # LSTM with 2048 hidden units
CLASSES = 101        # UCF101
LEN_MIN, LEN_MAX, LEN_MEAN, LEN_SD = 29, 1776, 187.0, 97.0


def sequence_lengths(rng: np.random.Generator, n: int) -> np.ndarray:
    """UCF101-shaped lengths: log-normal matched to mean 187 / sd 97, clipped."""
    var = np.log(1 + (LEN_SD / LEN_MEAN) ** 2)
    mu = np.log(LEN_MEAN) - var / 2
    return np.clip(rng.lognormal(mu, np.sqrt(var), size=n), LEN_MIN, LEN_MAX).astype(np.int64)


class VideoLSTM(torch.nn.Module):
    def __init__(self, features=FEATURES, hidden=HIDDEN, classes=CLASSES):
        super().__init__()
        self.lstm = torch.nn.LSTM(features, hidden, num_layers=1, batch_first=True)
        self.head = torch.nn.Linear(hidden, classes)

    def forward(self, x, lengths):
        # cuDNN's RNN path synchronises the device internally, which would wait
        # on the resident collective engine forever; torch's native LSTM
        # (cuBLAS GEMMs + fused cell kernels) does not
        with torch.backends.cudnn.flags(enabled=False):
            out, _ = self.lstm(x)
        last = out[torch.arange(x.shape[0], device=x.device), lengths - 1]
        return self.head(last)


def n_params(model: torch.nn.Module) -> int:
    return sum(p.numel() for p in model.parameters())


def bind_flat(model: torch.nn.Module, w: torch.Tensor, grad_bucket: torch.Tensor) -> None:
    """Make every parameter a view into the flat weights `w` and every .grad a
    view into the registered gradient bucket (same offsets)."""
    off = 0
    with torch.no_grad():
        for p in model.parameters():
            k = p.numel()
            w[off:off + k].copy_(p.reshape(-1))
            p.data = w[off:off + k].view_as(p)
            p.grad = grad_bucket[off:off + k].view_as(p)
            off += k
    assert off == w.numel() == grad_bucket.numel()


class SyntheticUCF101:
    """Per-(rank, step) deterministic batches with UCF101-shaped lengths."""

    def __init__(self, batch: int = 16, seed: int = 7, device=None, max_len: int | None = None):
        self.batch = batch
        self.seed = seed
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.max_len = max_len

    def batch_for(self, rank: int, step: int):
        rng = np.random.default_rng([self.seed, rank, step])
        lens = sequence_lengths(rng, self.batch)
        if self.max_len:
            lens = np.minimum(lens, self.max_len)
        T = int(lens.max())
        g = torch.Generator(device=self.device)
        g.manual_seed(int(rng.integers(1 << 62)))
        x = torch.randn(self.batch, T, FEATURES, device=self.device, generator=g)
        y = torch.randint(0, CLASSES, (self.batch,), device=self.device, generator=g)
        return x, torch.as_tensor(lens, device=self.device), y


def lstm_grad_step(model: VideoLSTM, bucket: torch.Tensor, batch):
    """Forward + backward accumulating into the registered bucket (fp32 with
    TF32 tensor cores); returns the loss tensor (left on the device)."""
    x, lens, y = batch
    bucket.zero_()
    logits = model(x, lens)
    loss = torch.nn.functional.cross_entropy(logits, y)
    with torch.backends.cudnn.flags(enabled=False):
        loss.backward()
    off = 0
    for p in model.parameters():   # autograd accumulates in place; re-home if it did not
        k = p.numel()
        view = bucket[off:off + k]
        if p.grad.data_ptr() != view.data_ptr():
            view.copy_(p.grad.reshape(-1))
            p.grad = view.view_as(p)
        off += k
    return loss
