"""Operator seam: drop-in for ``convkit.kernels`` (kernels.py:36-180).

Same six functions, same positional signatures, same in-place output
semantics, so the reference engine can be pointed at the GPU with

    import convkit.kernels, paper_1102_0183_b200.kernels as gpu
    for name in gpu.SEAM: setattr(convkit.kernels, name, getattr(gpu, name))

(the reference resolves ``kernels.<name>`` at call time, network.py:182-257;
its own fault-injection test swaps ``kernels.pull_bwd`` exactly this way).

Arguments may be numpy arrays (host: copied to the device, computed by the
CUDA kernel, copied back into the caller's arrays) or CUDA torch tensors
(used in place).  Every call runs the sm_100a kernel in ck_seam.cu; there is
no CPU path.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import ConfigError, DimensionError

ACT_SCALE = 1.7159
ACT_GAIN = 0.6666
SEAM = ("conv_fwd", "pull_bwd", "weight_grad", "bias_grad", "maxpool_fwd", "maxpool_bwd")

_workers = 1


def set_workers(n: int) -> None:
    """Accepted for API compatibility; the GPU kernels ignore it."""
    global _workers
    if n < 1:
        raise ConfigError(f"worker count must be >= 1, got {n}")
    _workers = int(n)


def get_workers() -> int:
    return _workers


def max_workers() -> int:
    return 1 << 16


class _Staged:
    """Device views of the call's arrays; numpy outputs are copied back."""

    def __init__(self):
        import torch
        if not torch.cuda.is_available():
            from .errors import StateError
            raise StateError("no CUDA device is visible (the seam has no CPU fallback)")
        self.torch = torch
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.writeback = []

    def __call__(self, arr, dtype=None, out=False):
        torch = self.torch
        if isinstance(arr, torch.Tensor):
            if not arr.is_cuda or not arr.is_contiguous():
                raise DimensionError("tensor arguments must be contiguous CUDA tensors")
            return arr
        host = np.asarray(arr)
        if dtype is not None and host.dtype != dtype:
            if out:
                raise DimensionError(f"output array must be {np.dtype(dtype).name}")
            host = host.astype(dtype)
        t = torch.from_numpy(np.ascontiguousarray(host)).to(self.dev)
        if out:
            self.writeback.append((arr, t))
        return t

    def stream(self):
        return self.torch.cuda.current_stream(self.dev).cuda_stream

    def finish(self):
        self.torch.cuda.current_stream(self.dev).synchronize()
        for host, t in self.writeback:
            host[...] = t.cpu().numpy()


def _shape3(t):
    if t.dim() != 3:
        raise DimensionError(f"expected a (maps, rows, pitch) stack, got shape {tuple(t.shape)}")
    return int(t.shape[0]), int(t.shape[1]), int(t.shape[2])


def conv_fwd(src, src_w, arena, fwd_offsets, fwd_srcs, fwd_widx, bias_off,
             kx, ky, sx, sy, a_out, y_out, out_w, out_h):
    s = _Staged()
    f32, i64 = np.float32, np.int64
    src_t = s(src, f32)
    a_t, y_t = s(a_out, f32, out=True), s(y_out, f32, out=True)
    tabs = [s(t, i64) for t in (fwd_offsets, fwd_srcs, fwd_widx, bias_off)]
    n_src, src_rows, src_pitch = _shape3(src_t)
    n_dest, out_rows, out_pitch = _shape3(a_t)
    _lib.call("ck_conv_fwd", src_t.data_ptr(), n_src, src_rows, src_pitch,
              s(arena, f32).data_ptr(), *[t.data_ptr() for t in tabs], kx, ky, sx, sy,
              a_t.data_ptr(), y_t.data_ptr(), n_dest, out_rows, out_pitch, out_w, out_h,
              s.stream())
    s.finish()


def pull_bwd(delta_next, dest_w, dest_h, arena, bwd_offsets, bwd_dests, bwd_widx,
             kx, ky, sx, sy, out, src_w, src_h):
    s = _Staged()
    f32, i64 = np.float32, np.int64
    d_t = s(delta_next, f32)
    o_t = s(out, f32, out=True)
    tabs = [s(t, i64) for t in (bwd_offsets, bwd_dests, bwd_widx)]
    n_dest, d_rows, d_pitch = _shape3(d_t)
    n_src, o_rows, o_pitch = _shape3(o_t)
    _lib.call("ck_pull_bwd", d_t.data_ptr(), n_dest, d_rows, d_pitch, dest_w, dest_h,
              s(arena, f32).data_ptr(), *[t.data_ptr() for t in tabs], kx, ky, sx, sy,
              o_t.data_ptr(), n_src, o_rows, o_pitch, src_w, src_h, s.stream())
    s.finish()


def weight_grad(delta_next, dest_w, dest_h, y_prev, pair_dest, pair_src, pair_off,
                kx, ky, sx, sy, g_arena):
    s = _Staged()
    f32, i64 = np.float32, np.int64
    d_t = s(delta_next, f32)
    y_t = s(y_prev, f32)
    g_t = s(g_arena, f32, out=True)
    tabs = [s(t, i64) for t in (pair_dest, pair_src, pair_off)]
    n_dest, d_rows, d_pitch = _shape3(d_t)
    n_src, y_rows, y_pitch = _shape3(y_t)
    _lib.call("ck_weight_grad", d_t.data_ptr(), n_dest, d_rows, d_pitch, dest_w, dest_h,
              y_t.data_ptr(), n_src, y_rows, y_pitch, *[t.data_ptr() for t in tabs],
              int(tabs[0].numel()), kx, ky, sx, sy, g_t.data_ptr(), s.stream())
    s.finish()


def bias_grad(delta_next, dest_w, dest_h, bias_off, g_arena):
    s = _Staged()
    d_t = s(delta_next, np.float32)
    g_t = s(g_arena, np.float32, out=True)
    b_t = s(bias_off, np.int64)
    n_dest, d_rows, d_pitch = _shape3(d_t)
    _lib.call("ck_bias_grad", d_t.data_ptr(), n_dest, d_rows, d_pitch, dest_w, dest_h,
              b_t.data_ptr(), g_t.data_ptr(), s.stream())
    s.finish()


def maxpool_fwd(src, px, py, out, out_w, out_h, arg_r, arg_c):
    s = _Staged()
    src_t = s(src, np.float32)
    o_t = s(out, np.float32, out=True)
    r_t, c_t = s(arg_r, np.int64, out=True), s(arg_c, np.int64, out=True)
    n, rows, pitch = _shape3(src_t)
    _, o_rows, o_pitch = _shape3(o_t)
    _lib.call("ck_maxpool_fwd", src_t.data_ptr(), n, rows, pitch, px, py, o_t.data_ptr(),
              o_rows, o_pitch, out_w, out_h, r_t.data_ptr(), c_t.data_ptr(), s.stream())
    s.finish()


def maxpool_bwd(delta_next, out_w, out_h, arg_r, arg_c, delta_prev):
    s = _Staged()
    d_t = s(delta_next, np.float32)
    p_t = s(delta_prev, np.float32, out=True)
    r_t, c_t = s(arg_r, np.int64), s(arg_c, np.int64)
    n, rows, pitch = _shape3(d_t)
    _, p_rows, p_pitch = _shape3(p_t)
    _lib.call("ck_maxpool_bwd", d_t.data_ptr(), n, rows, pitch, out_w, out_h,
              r_t.data_ptr(), c_t.data_ptr(), p_t.data_ptr(), p_rows, p_pitch, s.stream())
    s.finish()


def contrast(src, coeffs):
    """(C, rows, pitch) image stack and (F, fh, fw) f64 filters -> the (F*C)
    correlation maps (filters.py:168-172), dense (F*C, h, w) float32; the
    logical size is the stack's (rows, pitch)."""
    s = _Staged()
    src_t = s(src, np.float32)
    k = np.ascontiguousarray(coeffs, dtype=np.float64)
    k_t = s(k, np.float64)
    n, rows, pitch = _shape3(src_t)
    nf, fh, fw = k.shape
    out = s.torch.empty((nf * n, rows, pitch), dtype=s.torch.float32, device=s.dev)
    _lib.call("ck_contrast", src_t.data_ptr(), n, rows, pitch, pitch, rows, k_t.data_ptr(),
              nf, fh, fw, out.data_ptr(), rows, pitch, s.stream())
    s.torch.cuda.current_stream(s.dev).synchronize()
    return out.cpu().numpy()


# -- FC-side operators (inline numpy in the reference) --------------------------
# network.py:193-199 (forward), :209-230 (backward), :264-273 (update) and
# backprop.py:22-39 (output deltas, loss).  With these and the six kernels
# above every arithmetic step of NetworkState.train_step has a device entry.
FC_SEAM = ("fc_forward", "fc_backward", "act_deriv_mul", "sgd_update", "output_deltas")


def _vec(t):
    if t.dim() != 1:
        raise DimensionError(f"expected a vector, got shape {tuple(t.shape)}")
    return int(t.shape[0])


def fc_forward(x, weights, bias, a_out, y_out):
    """a = x @ W + b, y = activation(a) (network.py:197-199); W is (n_in, n_out)."""
    s = _Staged()
    f32 = np.float32
    x_t, w_t, b_t = s(x, f32), s(weights, f32), s(bias, f32)
    a_t = s(a_out, f32, out=True) if a_out is not None else None
    y_t = s(y_out, f32, out=True)
    n_in, n_out = _vec(x_t), _vec(b_t)
    if tuple(w_t.shape) != (n_in, n_out) or _vec(y_t) != n_out:
        raise DimensionError(f"FC shapes disagree: x {n_in}, W {tuple(w_t.shape)}, b {n_out}")
    _lib.call("ck_fc_fwd", x_t.data_ptr(), n_in, w_t.data_ptr(), b_t.data_ptr(), n_out,
              a_t.data_ptr() if a_t is not None else None, y_t.data_ptr(), s.stream())
    s.finish()


def fc_backward(x, weights, bias, delta, xgrad=None, grad_w=None, grad_b=None, eta=0.0):
    """xgrad = W @ delta (old W), grad_w = outer(x, delta), grad_b = delta
    (network.py:214-218); eta > 0 also applies the SGD step to W and b in
    place (network.py:271-273).  Outputs left as None are skipped."""
    if eta < 0:
        raise ConfigError(f"learning rate must be >= 0, got {eta}")
    s = _Staged()
    f32 = np.float32
    x_t, d_t = s(x, f32), s(delta, f32)
    upd = eta > 0
    w_t = s(weights, f32, out=upd)
    b_t = s(bias, f32, out=upd)
    xg = s(xgrad, f32, out=True) if xgrad is not None else None
    gw = s(grad_w, f32, out=True) if grad_w is not None else None
    gb = s(grad_b, f32, out=True) if grad_b is not None else None
    n_in, n_out = _vec(x_t), _vec(d_t)
    if tuple(w_t.shape) != (n_in, n_out) or _vec(b_t) != n_out:
        raise DimensionError(f"FC shapes disagree: x {n_in}, W {tuple(w_t.shape)}, "
                             f"delta {n_out}")
    ptr = (lambda t: t.data_ptr() if t is not None else None)
    _lib.call("ck_fc_bwd_update", x_t.data_ptr(), n_in, w_t.data_ptr(), b_t.data_ptr(), n_out,
              d_t.data_ptr(), ptr(xg), ptr(gw), ptr(gb), float(eta), s.stream())
    s.finish()


def act_deriv_mul(a, delta, width=None, height=None):
    """delta *= activation_deriv(a) (layers.py:28-30 as network.py:219/226/252
    apply it): a vector, or a (maps, rows, pitch) stack over its logical
    (width, height) cells (default: the whole stack)."""
    s = _Staged()
    a_t = s(a, np.float32)
    d_t = s(delta, np.float32, out=True)
    if tuple(a_t.shape) != tuple(d_t.shape):
        raise DimensionError(f"a {tuple(a_t.shape)} and delta {tuple(d_t.shape)} differ")
    if d_t.dim() == 1:
        maps, rows, pitch = 1, 1, int(d_t.shape[0])
    else:
        maps, rows, pitch = _shape3(d_t)
    w = pitch if width is None else int(width)
    h = rows if height is None else int(height)
    _lib.call("ck_act_deriv_mul", a_t.data_ptr(), d_t.data_ptr(), maps, rows, pitch, w, h,
              s.stream())
    s.finish()


def sgd_update(params, grads, eta):
    """params -= eta * grads in float32 (network.py:268-273)."""
    if eta <= 0:
        raise ConfigError(f"learning rate must be > 0, got {eta}")
    s = _Staged()
    p_t = s(params, np.float32, out=True)
    g_t = s(grads, np.float32)
    if p_t.numel() != g_t.numel():
        raise DimensionError(f"{p_t.numel()} parameters vs {g_t.numel()} gradients")
    _lib.call("ck_sgd_update", p_t.data_ptr(), g_t.data_ptr(), int(p_t.numel()), float(eta),
              s.stream())
    s.finish()


def output_deltas(y, targets, a, delta_out):
    """delta = (y - t) * f'(a) in float64 rounded to float32 (backprop.py:22-32);
    returns sample_loss(y, t) (backprop.py:35-39)."""
    s = _Staged()
    y_t, a_t = s(y, np.float32), s(a, np.float32)
    t_t = s(targets, np.float64)
    d_t = s(delta_out, np.float32, out=True)
    n = _vec(y_t)
    if _vec(t_t) != n or _vec(a_t) != n or _vec(d_t) != n:
        raise DimensionError("outputs, targets and deltas must have the same length")
    torch = s.torch
    loss = torch.zeros(1, dtype=torch.float64, device=s.dev)
    scratch = torch.empty(n, dtype=torch.float64, device=s.dev)
    _lib.call("ck_output_deltas", y_t.data_ptr(), a_t.data_ptr(), t_t.data_ptr(), n,
              d_t.data_ptr(), loss.data_ptr(), scratch.data_ptr(), s.stream())
    s.finish()
    return float(loss.item())
