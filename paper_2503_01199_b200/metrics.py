"""Training loss on the device: (1 - lambda) L1 + lambda (1 - SSIM) and its
analytic image gradient, plus PSNR / SSIM.

Reference: pkg/src/tinysplat/metrics.py:18-132 (float64 with scipy's
correlate1d, 11x11 Gaussian window sigma 1.5, valid interior, adjoint by
zero-embedding).  `loss_and_grad` runs the fused CUDA kernel
(sb_loss_fwd_bwd, one pass over the image); the separable torch conv2d
restatement below (`loss_and_grad_torch`) is kept as an independent check.
"""
from __future__ import annotations

import math

import torch
import torch.nn.functional as F

SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
C1 = 0.01 ** 2
C2 = 0.03 ** 2

_win_cache: dict = {}


def gaussian_window(size: int = SSIM_WINDOW, sigma: float = SSIM_SIGMA, device="cpu", dtype=torch.float64):
    x = torch.arange(size, dtype=torch.float64) - (size - 1) / 2.0
    w = torch.exp(-0.5 * (x / sigma) ** 2)
    return (w / w.sum()).to(device=device, dtype=dtype)


def _win(device, dtype):
    key = (str(device), dtype)
    if key not in _win_cache:
        w = gaussian_window(device=device, dtype=dtype)
        _win_cache[key] = (w.view(1, 1, -1, 1), w.view(1, 1, 1, -1))
    return _win_cache[key]


def _filter_valid(img, wc, wr):
    """(B, 1, H, W) -> (B, 1, H-10, W-10): correlate along rows then columns."""
    return F.conv2d(F.conv2d(img, wc), wr)


def _filter_transpose(field, wc, wr):
    """Adjoint of _filter_valid: embed the interior and correlate with zero padding."""
    r = wc.shape[2] // 2
    return F.conv2d(F.conv2d(F.pad(field, (r, r, r, r)), wc, padding=(r, 0)), wr, padding=(0, r))


def _ssim_terms(x, y, need_grad):
    wc, wr = _win(x.device, x.dtype)
    mu_x = _filter_valid(x, wc, wr)
    mu_y = _filter_valid(y, wc, wr)
    xx = _filter_valid(x * x, wc, wr)
    yy = _filter_valid(y * y, wc, wr)
    xy = _filter_valid(x * y, wc, wr)
    var_x, var_y, cov = xx - mu_x * mu_x, yy - mu_y * mu_y, xy - mu_x * mu_y
    A1 = 2.0 * mu_x * mu_y + C1
    A2 = 2.0 * cov + C2
    B1 = mu_x * mu_x + mu_y * mu_y + C1
    B2 = var_x + var_y + C2
    S = (A1 * A2) / (B1 * B2)
    per_ch = S.mean(dim=(1, 2, 3))
    if not need_grad:
        return per_ch, None
    n = S[0].numel()
    dA1 = A2 / (B1 * B2)
    dA2 = A1 / (B1 * B2)
    dB1 = -S / B1
    dB2 = -S / B2
    g_mu = 2.0 * mu_y * dA1 - 2.0 * mu_y * dA2 + 2.0 * mu_x * dB1 - 2.0 * mu_x * dB2
    grad = _filter_transpose(g_mu, wc, wr)
    grad = grad + _filter_transpose(2.0 * dA2, wc, wr) * y
    grad = grad + _filter_transpose(dB2, wc, wr) * (2.0 * x)
    return per_ch, grad / n


def _chw(img):
    return img.permute(2, 0, 1).unsqueeze(1)   # (H, W, C) -> (C, 1, H, W)


def ssim(a, b) -> float:
    a = torch.as_tensor(a)
    b = torch.as_tensor(b, device=a.device, dtype=a.dtype)
    if a.dim() == 2:
        a, b = a[..., None], b[..., None]
    vals, _ = _ssim_terms(_chw(a), _chw(b), False)
    return float(vals.mean())


def psnr(a, b) -> float:
    a = torch.as_tensor(a).double()
    b = torch.as_tensor(b, device=a.device).double()
    mse = float(((a - b) ** 2).mean())
    return math.inf if mse == 0.0 else 10.0 * math.log10(1.0 / mse)


def loss_and_grad(rendered: torch.Tensor, target, lam: float, return_tensor: bool = False, loss_out=None,
                  sse_out=None):
    """(loss, dL/d rendered) for (H, W, 3) images (metrics.py:118-132), fused
    kernel.  `target` may be float (any dtype) or uint8 (value / 255).  With
    return_tensor=True the loss stays a 0-d float64 device tensor (no sync).
    `loss_out`: a 1-element float64 tensor in pinned host memory that the
    kernel writes directly (mapped, zero-copy; no device-to-host copy in the
    stream) -- valid once the stream has reached this point; returned as the
    loss tensor with return_tensor=True.  `sse_out`: a 1-element float64
    device tensor that receives the call's sum of squared errors
    sum((rendered - target)^2) in float64 (psnr's numerator, formed by the
    same kernel; a device-to-device copy, no host sync)."""
    import ctypes as C
    from . import _lib
    from .errors import ShapeMismatchError
    _lib.require_cuda(rendered)
    x = rendered.float().contiguous()
    H, W, nch = x.shape
    if nch != 3:
        raise ShapeMismatchError(f"expected (H, W, 3) images, got {tuple(x.shape)}")
    y = torch.as_tensor(target, device=x.device)
    if tuple(y.shape) != tuple(x.shape):
        raise ShapeMismatchError(f"loss shapes {tuple(x.shape)} vs {tuple(y.shape)}")
    y8 = None
    if y.dtype == torch.uint8:
        y8, y = y.contiguous(), None
    else:
        y = y.float().contiguous()
    grad = torch.empty_like(x)
    # ticket + per-CTA partials: zeroed once, the ticket left zeroed by the call
    acc = _lib.workspace("loss_accum", _lib.load().sb_loss_workspace_bytes(W, H), x.device)
    out_ptr = None
    if loss_out is not None:
        if loss_out.device.type != "cpu" or not loss_out.is_pinned() or loss_out.dtype != torch.float64:
            raise ValueError("loss_out must be a pinned host float64 tensor")
        addr = C.c_void_p()
        if _lib.load().sb_host_mapped_pointer(C.c_void_p(loss_out.data_ptr()), C.byref(addr)) == 0 and addr.value:
            out, out_ptr = loss_out, addr
    if out_ptr is None:
        out = torch.empty(1, dtype=torch.float64, device=x.device)
        out_ptr = _lib.ptr(out)
    _lib.call("sb_loss_fwd_bwd", _lib.ptr(x), _lib.ptr(y), _lib.ptr(y8), W, H, float(lam), _lib.ptr(grad),
              _lib.ptr(acc), out_ptr, C.c_void_p(_lib.stream_ptr(x.device)))
    if sse_out is not None:
        sse_out.copy_(acc[72:80].view(torch.float64))
    if loss_out is not None and out is not loss_out:
        loss_out.copy_(out, non_blocking=True)   # not mappable: an async copy instead
        out = loss_out
    loss = out[0]
    return (loss if return_tensor else float(loss)), grad


def loss_and_grad_torch(rendered: torch.Tensor, target: torch.Tensor, lam: float, return_tensor: bool = False):
    """Separable-conv2d restatement of metrics.py:118-132 (independent check
    of the fused kernel)."""
    x = rendered.float()
    y = torch.as_tensor(target, device=x.device).float()
    diff = x - y
    nel = diff.numel()
    loss = (1.0 - lam) * diff.abs().mean()
    grad = torch.sign(diff) * ((1.0 - lam) / nel)
    if lam != 0.0:
        nch = x.shape[-1]
        vals, g = _ssim_terms(_chw(x), _chw(y), True)
        loss = loss + lam * (1.0 - vals.mean())
        grad = grad - lam * (g[:, 0].permute(1, 2, 0) / nch)
    return (loss if return_tensor else float(loss)), grad.contiguous()
