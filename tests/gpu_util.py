"""Helpers shared by the -m gpu parity tests (test infrastructure)."""
import numpy as np
import torch


def z14(X_gpu, X_or, A):
    """SURVEY Z14 parity metric: ||X_gpu - X_or||_F / max(||X_or||_F, 1e-3 ||A||_F)."""
    Xg = X_gpu.double().cpu().numpy() if torch.is_tensor(X_gpu) else np.asarray(X_gpu)
    An = np.linalg.norm(A.double().cpu().numpy() if torch.is_tensor(A) else A)
    den = max(np.linalg.norm(X_or), 1e-3 * An)
    return np.linalg.norm(Xg - X_or) / den


def cm(x, dtype, device="cuda"):
    """column-major device copy"""
    t = torch.as_tensor(np.asarray(x)) if not torch.is_tensor(x) else x
    return t.to(device=device, dtype=dtype).t().contiguous().t()


def np64(t):
    return t.double().cpu().numpy()
