"""Helpers for the GPU parity tests: move numpy arrays to/from CUDA as bit
patterns (int32/int64 views, so no unsigned-dtype kernel support is needed)."""
import numpy as np
import torch

_VIEW = {np.dtype(np.uint32): np.int32, np.dtype(np.uint64): np.int64}


def dev(a: np.ndarray) -> torch.Tensor:
    a = np.ascontiguousarray(a)
    return torch.from_numpy(a.view(_VIEW[a.dtype])).cuda()


def host(t: torch.Tensor, dt) -> np.ndarray:
    return t.cpu().numpy().view(dt)


def free_host_gb() -> float:
    try:
        import psutil
        return psutil.virtual_memory().available / 2 ** 30
    except Exception:
        return 0.0


def free_dev_gb() -> float:
    f, _ = torch.cuda.mem_get_info()
    return f / 2 ** 30
