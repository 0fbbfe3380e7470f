"""Datasets and the per-epoch batch schedule (src/store.py:21-81).

On the B200 path a dataset is uploaded to HBM once (``Trainer`` does it,
deduplicated by content hash) and each model indexes it through its own
epoch permutation; :func:`batches` is kept for host-side callers and for
the e2e host-fed step, with the reference's exact semantics.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

from . import formats, rng


@dataclass(frozen=True)
class Dataset:
    content_hash: str
    train_x: np.ndarray
    train_y: np.ndarray
    test_x: np.ndarray
    test_y: np.ndarray

    @property
    def sample_count(self) -> int:
        return int(self.train_x.shape[0])

    @property
    def nbytes(self) -> int:
        return int(self.train_x.nbytes + self.train_y.nbytes + self.test_x.nbytes + self.test_y.nbytes)

    @property
    def sample_shape(self) -> tuple:
        return tuple(self.train_x.shape[1:])


@dataclass(frozen=True)
class Batch:
    x: np.ndarray
    y: np.ndarray


def content_hash(blob: bytes) -> str:
    return hashlib.sha256(blob).hexdigest()


def decode(blob: bytes) -> Dataset:
    return Dataset(content_hash=content_hash(blob), **formats.decode_dataset(blob))


def from_splits(splits: dict) -> Dataset:
    """Encode once to fix the content hash, keep the arrays as given."""
    blob = formats.encode_dataset(splits)
    return Dataset(
        content_hash(blob),
        *(np.ascontiguousarray(splits[k], dtype=np.float32) for k in formats.DATASET_SECTIONS),
    )


def batch_count(samples: int, batch_size: int) -> int:
    return -(-samples // batch_size)


def epoch_permutation(dataset: Dataset, job_seed: int, epoch: int) -> np.ndarray:
    """The keyed shuffle of one epoch (src/store.py:74-76)."""
    return rng.permutation(dataset.sample_count, "shuffle", dataset.content_hash, job_seed, epoch)


def batches(dataset: Dataset, batch_size: int, job_seed: int, epoch: int) -> list:
    perm = epoch_permutation(dataset, job_seed, epoch)
    return [
        Batch(dataset.train_x[perm[s:s + batch_size]], dataset.train_y[perm[s:s + batch_size]])
        for s in range(0, dataset.sample_count, batch_size)
    ]
