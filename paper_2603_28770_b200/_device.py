"""Device plumbing: PyTorch owns device memory and streams; kernels are ours."""

from __future__ import annotations

import numpy as np
import torch

from ._capi import ZeusNativeError, lib

F64 = torch.float64


def require_device(device=None) -> torch.device:
    """The CUDA device the call runs on.  No CPU fallback: raises if absent."""
    if not torch.cuda.is_available():
        raise ZeusNativeError("no CUDA device visible; paper_2603_28770_b200 runs only on B200")
    lib()  # fail loudly if the extension is missing
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ZeusNativeError(f"device {dev} is not a CUDA device")
    return dev if dev.index is not None else torch.device("cuda", torch.cuda.current_device())


def stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def empty(shape, device, dtype=F64) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=device)


def workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device)


def to_soa(points: np.ndarray, device) -> torch.Tensor:
    """[n][d] host points -> SoA [d][n] float64 device tensor."""
    arr = np.ascontiguousarray(np.asarray(points, dtype=np.float64).T)
    return torch.from_numpy(arr).to(device)


def from_soa(t: torch.Tensor) -> np.ndarray:
    """SoA [d][n] device tensor -> [n][d] host array."""
    return np.ascontiguousarray(t.cpu().numpy().T)
