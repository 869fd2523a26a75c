"""CPU restatement of the reference training glue (test infrastructure only).

Checker for paper_2111_00110_b200/trainer.py; pinned to the reference's own
outputs in tests/golden/trainer.npz (tests/golden/make_golden_trainer.py).
Follows reference trainer.py:70-152 (losses, L1 term, SGD/Adam step with
bias correction and domain clipping).  Only tests/ may import this module.
"""

from __future__ import annotations

import numpy as np

DOMAIN_MARGIN = 1e-6


def loss_and_tangent(pred, target, loss, mask=None):
    """trainer.py:70-105."""
    diff = np.asarray(pred, np.float64) - np.asarray(target, np.float64)
    if mask is not None:
        mk = np.reshape(mask, np.shape(mask) + (1,) * (diff.ndim - np.ndim(mask)))
        diff = np.where(mk, diff, 0.0)
        count = int(np.sum(mask)) * (diff.size // np.size(mask))
    else:
        count = diff.size
    if count == 0:
        return 0.0, np.zeros_like(diff)
    if loss == "mae":
        return float(np.abs(diff).sum()) / count, np.sign(diff) / count
    return float((diff * diff).sum()) / count, 2.0 * diff / count


def l1_term(w, lam):
    """trainer.py:108-112."""
    w = np.asarray(w, np.float64)
    if lam == 0.0:
        return 0.0, np.zeros_like(w)
    return lam * float(np.abs(w).sum()), lam * np.sign(w)


class Optimizer:
    """trainer.py:115-152: SGD / Adam (0.9, 0.999, 1e-8) over (w, p, bias)."""

    def __init__(self, optimizer="adam", lr=1e-2, schedule=(), train_positions=True):
        self.kind, self.lr, self.schedule = optimizer, lr, sorted(schedule)
        self.train_positions = train_positions
        self.t, self.m, self.v = 0, {}, {}

    def lr_at(self, epoch):
        lr = self.lr
        for start, value in self.schedule:
            if epoch >= start:
                lr = value
        return lr

    def _dir(self, name, g):
        if self.kind == "sgd":
            return g
        m = self.m.setdefault(name, np.zeros_like(g))
        v = self.v.setdefault(name, np.zeros_like(g))
        m += 0.1 * (g - m)
        v += 0.001 * (g * g - v)
        return (m / (1 - 0.9 ** self.t)) / (np.sqrt(v / (1 - 0.999 ** self.t)) + 1e-8)

    def step(self, p, w, w_bar, p_bar, epoch, bias=0.0, bias_bar=None):
        if not np.all(np.isfinite(w_bar)) or (p_bar is not None and not np.all(np.isfinite(p_bar))):
            raise FloatingPointError("non-finite gradient in optimizer step")
        self.t += 1
        lr = self.lr_at(epoch)
        w = w - lr * self._dir("w", np.asarray(w_bar, np.float64))
        if p_bar is not None and self.train_positions:
            p = np.clip(p - lr * self._dir("p", np.asarray(p_bar, np.float64)),
                        -1.0 + DOMAIN_MARGIN, 1.0 - DOMAIN_MARGIN)
        if bias_bar is not None:
            bias = bias - lr * float(self._dir("bias", np.array([bias_bar]))[0])
        return p, w, bias
