"""Shared helpers for the GPU parity tests (seeded inputs, oracle wiring)."""
from __future__ import annotations

import numpy as np
import torch

import oracle


def sym_bf16(seed: int, shape) -> torch.Tensor:
    """Uniform [-1, 1) from the portable synth::Rng mapping (synth.cpp:24-29), rounded to bf16."""
    n = int(np.prod(shape))
    x = oracle.fill_symmetric(seed, 1.0, n).reshape(shape)
    return torch.from_numpy(x).to(torch.bfloat16)


def bf16_to_f64(t: torch.Tensor) -> np.ndarray:
    return t.float().cpu().numpy().astype(np.float64)


# max-abs error / tolerance of every numeric parity check, printed in pytest's terminal summary
MARGINS: list[tuple[str, float, float]] = []


def record_margin(name: str, err: float, tol: float) -> None:
    MARGINS.append((name, float(err), float(tol)))
