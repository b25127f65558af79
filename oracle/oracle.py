"""CPU oracle of the online-BP hot path (TEST INFRASTRUCTURE ONLY).

Restates the reference (convkit, /root/reference/pkg/src/convkit) on the
host: the six numba kernels and the contrast correlation come from
``liboracle.so`` (ck_oracle.c, same arithmetic as kernels.py), and the
network walk below follows ``network.py`` line by line, using numpy for the
FC layers, activations and updates exactly as the reference does (OpenBLAS
sgemv, numpy float32 tanh, NEP-50 weak scalars).  On one host it therefore
reproduces the reference bit for bit; pinned by tests/test_oracle_golden.py
against fixtures produced by the reference itself (tests/golden/make_golden.py).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may use this
module — never the product path.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

ACT_SCALE = 1.7159
ACT_GAIN = 0.6666

_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        I = C.c_int
        I64 = C.c_int64
        L.oracle_conv_fwd.argtypes = [P, I64, I64, P, P, P, P, P, I, I, I, I, P, P, I,
                                      I64, I64, I, I]
        L.oracle_pull_bwd.argtypes = [P, I64, I64, I, I, P, P, P, P, I, I, I, I, P, I,
                                      I64, I64, I, I]
        L.oracle_weight_grad.argtypes = [P, I64, I64, I, I, P, I64, I64, P, P, P, I, I, I,
                                         I, I, P]
        L.oracle_bias_grad.argtypes = [P, I64, I64, I, I, I, P, P]
        L.oracle_maxpool_fwd.argtypes = [P, I64, I64, I, I, P, I64, I64, I, I, I, P, P]
        L.oracle_maxpool_bwd.argtypes = [P, I64, I64, I, I, I, P, P, P, I64, I64]
        L.oracle_contrast.argtypes = [P, I, I64, I64, I, I, P, I, I, I, P, I64, I64]
        L.oracle_set_threads.argtypes = [I]
        L.oracle_get_threads.restype = I
        for f in ("oracle_conv_fwd", "oracle_pull_bwd", "oracle_weight_grad",
                  "oracle_bias_grad", "oracle_maxpool_fwd", "oracle_maxpool_bwd",
                  "oracle_contrast", "oracle_set_threads"):
            getattr(L, f).restype = None
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def get_threads() -> int:
    return int(lib().oracle_get_threads())


def _p(a: np.ndarray):
    assert a.flags.c_contiguous, "oracle buffers must be C-contiguous"
    return a.ctypes.data


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


# -- the six kernels with convkit.kernels signatures (pitched numpy arrays) --

def conv_fwd(src, src_w, arena, fwd_offsets, fwd_srcs, fwd_widx, bias_off,
             kx, ky, sx, sy, a_out, y_out, out_w, out_h):
    tabs = [_i64(t) for t in (fwd_offsets, fwd_srcs, fwd_widx, bias_off)]
    lib().oracle_conv_fwd(_p(src), src.shape[1] * src.shape[2], src.shape[2], _p(arena),
                          *map(_p, tabs), kx, ky, sx, sy, _p(a_out), _p(y_out),
                          a_out.shape[0], a_out.shape[1] * a_out.shape[2], a_out.shape[2],
                          out_w, out_h)


def pull_bwd(delta_next, dest_w, dest_h, arena, bwd_offsets, bwd_dests, bwd_widx,
             kx, ky, sx, sy, out, src_w, src_h):
    tabs = [_i64(t) for t in (bwd_offsets, bwd_dests, bwd_widx)]
    lib().oracle_pull_bwd(_p(delta_next), delta_next.shape[1] * delta_next.shape[2],
                          delta_next.shape[2], dest_w, dest_h, _p(arena), *map(_p, tabs),
                          kx, ky, sx, sy, _p(out), out.shape[0],
                          out.shape[1] * out.shape[2], out.shape[2], src_w, src_h)


def weight_grad(delta_next, dest_w, dest_h, y_prev, pair_dest, pair_src, pair_off,
                kx, ky, sx, sy, g_arena):
    tabs = [_i64(t) for t in (pair_dest, pair_src, pair_off)]
    lib().oracle_weight_grad(_p(delta_next), delta_next.shape[1] * delta_next.shape[2],
                             delta_next.shape[2], dest_w, dest_h, _p(y_prev),
                             y_prev.shape[1] * y_prev.shape[2], y_prev.shape[2],
                             *map(_p, tabs), len(tabs[0]), kx, ky, sx, sy, _p(g_arena))


def bias_grad(delta_next, dest_w, dest_h, bias_off, g_arena):
    b = _i64(bias_off)
    lib().oracle_bias_grad(_p(delta_next), delta_next.shape[1] * delta_next.shape[2],
                           delta_next.shape[2], dest_w, dest_h, delta_next.shape[0],
                           _p(b), _p(g_arena))


def maxpool_fwd(src, px, py, out, out_w, out_h, arg_r, arg_c):
    lib().oracle_maxpool_fwd(_p(src), src.shape[1] * src.shape[2], src.shape[2], px, py,
                             _p(out), out.shape[1] * out.shape[2], out.shape[2], out_w,
                             out_h, src.shape[0], _p(arg_r), _p(arg_c))


def maxpool_bwd(delta_next, out_w, out_h, arg_r, arg_c, delta_prev):
    lib().oracle_maxpool_bwd(_p(delta_next), delta_next.shape[1] * delta_next.shape[2],
                             delta_next.shape[2], out_w, out_h, delta_next.shape[0],
                             _p(arg_r), _p(arg_c), _p(delta_prev),
                             delta_prev.shape[1] * delta_prev.shape[2], delta_prev.shape[2])


def contrast(src: np.ndarray, coeffs: np.ndarray) -> np.ndarray:
    """(C, H, W) f32 image, (F, fh, fw) f64 filters -> (F*C, H, W) responses."""
    src = np.ascontiguousarray(src, dtype=np.float32)
    coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
    n_ch, h, w = src.shape
    nf, fh, fw = coeffs.shape
    out = np.zeros((nf * n_ch, h, w), dtype=np.float32)
    lib().oracle_contrast(_p(src), n_ch, h * w, w, w, h, _p(coeffs), nf, fh, fw,
                          _p(out), h * w, w)
    return out


# -- numpy restatement of layers.py / backprop.py -----------------------

def activation(a):
    return ACT_SCALE * np.tanh(ACT_GAIN * a)


def activation_deriv(a):
    t = np.tanh(ACT_GAIN * a)
    return ACT_SCALE * ACT_GAIN * (1.0 - t * t)


def output_deltas(outputs, targets, pre):
    return (np.asarray(outputs) - np.asarray(targets)) * activation_deriv(np.asarray(pre))


def sample_loss(outputs, targets) -> float:
    o = np.asarray(outputs, dtype=np.float64)
    t = np.asarray(targets, dtype=np.float64)
    return 0.5 * float(((o - t) ** 2).sum())


# -- network walk (network.py:163-286) ----------------------------------

class _L:
    pass


class OracleNet:
    """CPU restatement of NetworkState for float32 nets.

    Built from a resolved NetworkSpec with the same tables and initial
    weights as the reference (the tables come from the product's host-side
    topology module, itself pinned against reference fixtures).  Buffers are
    dense (maps, h, w); the reference proves pitch does not change results
    (tests/test_network.py:58-69 in the reference).
    """

    def __init__(self, spec, seed, table_seed=0x7AB1E, params=None):
        from paper_1102_0183_b200.network import _padded_bank
        from paper_1102_0183_b200.topology import build_full_table, build_random_table

        self.spec = spec
        self.layers = []
        f32 = np.float32
        for idx, ls in enumerate(spec.layers):
            prev = spec.layers[idx - 1] if idx else None
            L = _L()
            L.kind = ls.kind
            if ls.is_spatial:
                shape = (ls.out_maps, ls.out_height, ls.out_width)
                L.y = np.zeros(shape, f32)
            if ls.kind == "input":
                L.delta = None
            elif ls.kind == "image_processing":
                L.coeffs, _, _ = _padded_bank(ls.filters)
                L.delta = None
            elif ls.kind == "convolutional":
                if ls.connectivity == "random":
                    L.table = build_random_table(prev.out_maps, ls.maps, ls.in_degree,
                                                 [table_seed, idx], ls.kernel)
                else:
                    L.table = build_full_table(prev.out_maps, ls.maps, ls.kernel)
                L.skip = ls.skip
                L.arena = np.zeros(L.table.arena_size, f32)
                L.a = np.zeros(shape, f32)
                L.delta = np.zeros(shape, f32)
                L.grad = np.zeros_like(L.arena)
            elif ls.kind == "max_pooling":
                L.region = ls.pool
                L.delta = np.zeros(shape, f32)
                L.arg_r = np.zeros(shape, np.int64)
                L.arg_c = np.zeros(shape, np.int64)
            else:
                n_in = (prev.out_maps * prev.out_width * prev.out_height
                        if prev.is_spatial else prev.neurons)
                L.weights = np.zeros((n_in, ls.neurons), f32)
                L.bias = np.zeros(ls.neurons, f32)
                L.a = np.zeros(ls.neurons, f32)
                L.y = np.zeros(ls.neurons, f32)
                L.delta = np.zeros(ls.neurons, f32)
                L.x = np.zeros(n_in, f32)
                L.grad_w = np.zeros_like(L.weights)
                L.grad_b = np.zeros_like(L.bias)
            self.layers.append(L)
        rng = np.random.default_rng(seed)
        for L in self.layers:
            if L.kind == "convolutional":
                L.arena[:] = rng.uniform(-0.05, 0.05, L.arena.shape)
            elif L.kind in ("fully_connected", "output"):
                L.weights[:] = rng.uniform(-0.05, 0.05, L.weights.shape)
                L.bias[:] = rng.uniform(-0.05, 0.05, L.bias.shape)
        if params is not None:
            self.set_flat_parameters(params)

    def parameters(self):
        for idx, L in enumerate(self.layers):
            if L.kind == "convolutional":
                yield idx, "arena", L.arena
            elif L.kind in ("fully_connected", "output"):
                yield idx, "weights", L.weights
                yield idx, "bias", L.bias

    def flat_parameters(self) -> np.ndarray:
        return np.concatenate([a.ravel() for _, _, a in self.parameters()])

    def set_flat_parameters(self, flat) -> None:
        flat = np.asarray(flat, dtype=np.float32)
        off = 0
        for _, _, a in self.parameters():
            a[...] = flat[off:off + a.size].reshape(a.shape)
            off += a.size

    def forward(self, channels):
        first = self.layers[0]
        first.y[:] = channels
        prev = first
        for L in self.layers[1:]:
            if L.kind == "image_processing":
                resp = contrast(prev.y, L.coeffs)
                c = prev.y.shape[0]
                L.y[:c] = prev.y
                L.y[c:] = resp
            elif L.kind == "convolutional":
                t = L.table
                conv_fwd(prev.y, prev.y.shape[2], L.arena, t._fwd_offsets, t._fwd_srcs,
                         t._fwd_widx, t.bias_offset, t.kx, t.ky, L.skip[0], L.skip[1],
                         L.a, L.y, L.y.shape[2], L.y.shape[1])
            elif L.kind == "max_pooling":
                maxpool_fwd(prev.y, L.region[0], L.region[1], L.y, L.y.shape[2],
                            L.y.shape[1], L.arg_r, L.arg_c)
            else:
                if prev.kind in ("fully_connected", "output"):
                    L.x[:] = prev.y
                else:
                    L.x[:] = prev.y.ravel()
                L.a[:] = L.x @ L.weights + L.bias
                L.y[:] = activation(L.a)
            prev = L
        return self.layers[-1].y

    def backward(self, targets):
        layers = self.layers
        k = len(layers) - 1
        out = layers[k]
        out.delta[:] = output_deltas(out.y, targets, out.a)
        while layers[k].kind in ("fully_connected", "output"):
            fc = layers[k]
            np.outer(fc.x, fc.delta, out=fc.grad_w)
            fc.grad_b[:] = fc.delta
            xgrad = fc.weights @ fc.delta
            k -= 1
            below = layers[k]
            if below.kind in ("fully_connected", "output"):
                below.delta[:] = xgrad * activation_deriv(below.a)
            elif below.delta is not None:
                below.delta[:] = xgrad.reshape(below.delta.shape)
                if below.kind == "convolutional":
                    below.delta[:] *= activation_deriv(below.a)
            else:
                return
        while k >= 1:
            L = layers[k]
            prev = layers[k - 1]
            if L.kind == "convolutional":
                t = L.table
                dh, dw = L.delta.shape[1], L.delta.shape[2]
                weight_grad(L.delta, dw, dh, prev.y, t._pair_dest, t._pair_src,
                            t.pair_offsets, t.kx, t.ky, L.skip[0], L.skip[1], L.grad)
                bias_grad(L.delta, dw, dh, t.bias_offset, L.grad)
                if prev.delta is None:
                    return
                pull_bwd(L.delta, dw, dh, L.arena, t._bwd_offsets, t._bwd_dests,
                         t._bwd_widx, t.kx, t.ky, L.skip[0], L.skip[1], prev.delta,
                         prev.delta.shape[2], prev.delta.shape[1])
            else:
                if prev.delta is None:
                    return
                prev.delta[:] = 0
                maxpool_bwd(L.delta, L.delta.shape[2], L.delta.shape[1], L.arg_r, L.arg_c,
                            prev.delta)
            if prev.kind == "convolutional":
                prev.delta[:] *= activation_deriv(prev.a)
            k -= 1

    def apply_gradients(self, eta):
        for L in self.layers:
            if L.kind == "convolutional":
                L.arena -= eta * L.grad
            elif L.kind in ("fully_connected", "output"):
                L.weights -= eta * L.grad_w
                L.bias -= eta * L.grad_b

    def train_step(self, channels, targets, eta):
        out = self.forward(channels)
        loss = sample_loss(out, targets)
        self.backward(targets)
        if eta > 0:
            self.apply_gradients(eta)
        return loss

    def predict(self, channels) -> int:
        return int(np.argmax(self.forward(channels)))


def targets_for(label: int, n_classes: int) -> np.ndarray:
    t = np.full(n_classes, -1.0)
    t[label] = 1.0
    return t


def train_sequence(net: OracleNet, images_f32, labels, order, eta, n_classes):
    """training.train_epoch's inner loop over a given visit order; mean loss."""
    targets = np.eye(n_classes, dtype=np.float64) * 2.0 - 1.0
    total = 0.0
    for i in order:
        total += net.train_step(images_f32[i], targets[labels[i]], eta)
    return total / len(order)
