"""Device-buffer plumbing: torch CUDA tensors are used only as fp64 device
memory and stream handles for the C-ABI."""

import numpy as np
import torch

DEVICE = "cuda"


def as_dev(x):
    """fp64 contiguous CUDA tensor view/copy of x (numpy, list or tensor)."""
    if isinstance(x, torch.Tensor):
        t = x
        if t.device.type != "cuda":
            t = t.to(DEVICE)
        if t.dtype != torch.float64:
            t = t.to(torch.float64)
        return t.contiguous()
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device=DEVICE)


def empty_dev(n):
    return torch.empty(int(n), dtype=torch.float64, device=DEVICE)


def zeros_dev(n):
    return torch.zeros(int(n), dtype=torch.float64, device=DEVICE)


def ptr(t):
    return t.data_ptr() if t is not None else None


def stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def to_host(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)
