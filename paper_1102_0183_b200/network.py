"""Device-resident ``NetworkState`` (mirror of convkit ``network.py:81-304``).

Construction is the reference's: the same layer walk, the same seeded
connection tables (``[table_seed, layer_idx]``, network.py:103-108) and the
same weight initialisation order (``default_rng(seed).uniform(-0.05, 0.05)``
over each conv arena, then FC weights, then FC bias, network.py:128-136).
The resulting tables and parameters are uploaded once; every forward,
backward and update afterwards runs in the CUDA engine (ck_net.cu).

Differences from the reference, all deliberate:
  * FP32 only — ``dtype=float64`` raises PrecisionError (double nets are the
    CPU oracle's job).
  * ``forward`` returns a host copy of the outputs, not a live view.
  * layer buffers are read back on demand through ``layers[i]`` views.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .device import current_stream_handle
from .errors import ConfigError, DimensionError, PrecisionError, StateError
from .filters import expand_selection, filter_coefficients
from .topology import (ConnectionTable, NetworkSpec, build_full_table,
                       build_random_table)

DEFAULT_TABLE_SEED = 0x7AB1E
DEFAULT_PITCH_QUANTUM = 32

KIND_CODES = {"input": 0, "image_processing": 1, "convolutional": 2,
              "max_pooling": 3, "fully_connected": 4, "output": 4}
BUF_A, BUF_Y, BUF_DELTA, BUF_ARG, BUF_GRAD = range(5)
TEAM_AUTO, TEAM_CLUSTER, TEAM_GRID = range(3)


def _padded_bank(selection) -> tuple[np.ndarray, int, int]:
    """Expanded filters zero-padded (centred) to one common odd size; extra
    zero taps add exact zeros to the f64 sum, so results are unchanged."""
    coeffs = [filter_coefficients(n) for n in expand_selection(selection)]
    fh = max(c.shape[0] for c in coeffs)
    fw = max(c.shape[1] for c in coeffs)
    out = np.zeros((len(coeffs), fh, fw), dtype=np.float64)
    for i, c in enumerate(coeffs):
        oy, ox = (fh - c.shape[0]) // 2, (fw - c.shape[1]) // 2
        out[i, oy:oy + c.shape[0], ox:ox + c.shape[1]] = c
    return np.ascontiguousarray(out), fh, fw


class LayerView:
    """Read-only window onto one device layer (reference attribute names)."""

    def __init__(self, net: "NetworkState", idx: int, kind: str, shape, table=None,
                 region=None, skip=None, selection=None):
        self._net = net
        self.index = idx
        self.kind = kind
        self.shape = tuple(shape)          # (maps, h, w) or (neurons,)
        self.table = table
        self.region = region
        self.skip = skip
        self.selection = selection

    def _read(self, which, dtype=np.float32, shape=None):
        return self._net._read_buffer(self.index, which, dtype, shape or self.shape)

    @property
    def y(self) -> np.ndarray:
        return self._read(BUF_Y)

    @property
    def a(self) -> np.ndarray:
        return self._read(BUF_A)

    @property
    def delta(self) -> np.ndarray:
        return self._read(BUF_DELTA)

    def _arg(self):
        flat = self._read(BUF_ARG, np.int32)
        src = self._net.spec.layers[self.index - 1]
        local = flat % (src.out_height * src.out_width)
        return local // src.out_width, local % src.out_width

    @property
    def arg_r(self) -> np.ndarray:
        return self._arg()[0].astype(np.int64)

    @property
    def arg_c(self) -> np.ndarray:
        return self._arg()[1].astype(np.int64)

    @property
    def grad(self) -> np.ndarray:
        n = self._net._buffer_size(self.index, BUF_GRAD)
        return self._net._read_buffer(self.index, BUF_GRAD, np.float32, (n,))


def layer_descs(spec: NetworkSpec, table_seed: int = DEFAULT_TABLE_SEED):
    """The C-ABI description of a resolved net: (ck_layer_desc array, host
    arrays it points into, connection tables, parameter layout, parameter
    count).  Tables are the reference's: seeded ``[table_seed, layer_idx]``
    random tables (network.py:103-108) or full tables."""
    descs = (_lib.LayerDesc * len(spec.layers))()
    keep = []                            # host arrays alive while descs are used
    tables: dict[int, ConnectionTable] = {}
    layout: list[tuple[int, str, tuple, int]] = []
    offset = 0
    for idx, ls in enumerate(spec.layers):
        prev = spec.layers[idx - 1] if idx else None
        d = descs[idx]
        d.kind = KIND_CODES[ls.kind]
        d.maps, d.width, d.height = ls.out_maps, ls.out_width, ls.out_height
        if ls.kind == "image_processing":
            bank, fh, fw = _padded_bank(ls.filters)
            keep.append(bank)
            d.n_filters, d.filter_h, d.filter_w = bank.shape[0], fh, fw
            d.filter_coeffs = bank.ctypes.data
        elif ls.kind == "convolutional":
            if ls.connectivity == "random":
                table = build_random_table(prev.out_maps, ls.maps, ls.in_degree,
                                           [table_seed, idx], ls.kernel)
            else:
                table = build_full_table(prev.out_maps, ls.maps, ls.kernel)
            tables[idx] = table
            d.kx, d.ky = table.kx, table.ky
            d.sx, d.sy = ls.skip
            d.n_pairs = table.n_pairs
            d.arena_size = table.arena_size
            arrays = [np.ascontiguousarray(a, dtype=np.int64) for a in
                      (table._fwd_offsets, table._fwd_srcs, table._fwd_widx,
                       table.bias_offset)]
            keep.extend(arrays)
            d.fwd_offsets, d.fwd_srcs, d.fwd_widx, d.bias_offset = (
                a.ctypes.data for a in arrays)
            layout.append((idx, "arena", (table.arena_size,), offset))
            offset += table.arena_size
        elif ls.kind == "max_pooling":
            d.px, d.py = ls.pool
        elif ls.kind in ("fully_connected", "output"):
            n_in = (prev.out_maps * prev.out_width * prev.out_height
                    if prev.is_spatial else prev.neurons)
            layout.append((idx, "weights", (n_in, ls.neurons), offset))
            offset += n_in * ls.neurons
            layout.append((idx, "bias", (ls.neurons,), offset))
            offset += ls.neurons
    return descs, keep, tables, layout, offset


class NetworkState:
    """All weights plus device scratch state for one network instance."""

    def __init__(self, spec: NetworkSpec, seed: int, dtype=None,
                 pitch_quantum: int = DEFAULT_PITCH_QUANTUM,
                 table_seed: int = DEFAULT_TABLE_SEED, device: int = 0,
                 team: tuple[int, int, int] | None = None):
        self.spec = spec
        self.seed = seed
        self.table_seed = table_seed
        self.dtype = np.dtype(dtype) if dtype is not None else np.dtype(np.float32)
        if self.dtype != np.float32:
            raise PrecisionError(
                f"the B200 engine computes in float32 only, got {self.dtype}")
        self.pitch_quantum = pitch_quantum
        self.device = device
        self._handle = None
        self.tables: dict[int, ConnectionTable] = {}
        self._param_layout: list[tuple[int, str, tuple, int]] = []

        descs, keep, self.tables, self._param_layout, self._n_params = layer_descs(
            spec, table_seed)
        self.layers: list[LayerView] = []
        for idx, ls in enumerate(spec.layers):
            if ls.is_spatial:
                shape = (ls.out_maps, ls.out_height, ls.out_width)
            else:
                shape = (ls.neurons,)
            self.layers.append(LayerView(self, idx, ls.kind, shape, self.tables.get(idx),
                                         ls.pool if ls.kind == "max_pooling" else None,
                                         ls.skip if ls.kind == "convolutional" else None,
                                         ls.filters or None))

        self._descs, self._desc_keep = descs, keep     # reused by the tensor-core eval plan
        self._tc_plans: dict = {}
        self._tc_loaded: dict = {}     # plan key -> self._version its weights reflect
        self._version = 0
        handle = C.c_void_p()
        _lib.call("ck_net_create", descs, len(spec.layers), device, C.byref(handle))
        self._handle = handle
        n = C.c_int64()
        _lib.call("ck_net_num_params", self._handle, C.byref(n))
        if n.value != self._n_params:
            raise StateError(f"engine holds {n.value} parameters, expected {self._n_params}")
        if team is not None:
            self.set_team(*team)
        self._init_weights(seed)

    # -- lifecycle -----------------------------------------------------

    def tc_plan(self, passes: int = 3, max_batch: int = 4096):
        """Tensor-core evaluation plan (ck_tc_create) for this net's geometry,
        loaded with the current parameters."""
        key = (passes, max_batch)
        plan = self._tc_plans.get(key)
        if plan is None:
            plan = C.c_void_p()
            _lib.call("ck_tc_create", self._descs, len(self.spec.layers), self.device,
                      max_batch, passes, C.byref(plan))
            self._tc_plans[key] = plan
        if self._tc_loaded.get(key) != self._version:
            if self._handle is None:
                raise StateError("network has been closed")
            params = C.c_void_p()
            _lib.call("ck_net_device_params", self._handle, C.byref(params))
            _lib.call("ck_tc_set_params", plan, params, current_stream_handle(self.device))
            self._tc_loaded[key] = self._version
        return plan

    def tct_plan(self):
        """Tensor-core TRAINING plan (ck_tct_create) over this
        net's device parameters: it trains them in place."""
        plan = getattr(self, "_tct_plan", None)
        if plan is None:
            params = C.c_void_p()
            _lib.call("ck_net_device_params", self.handle, C.byref(params))
            plan = C.c_void_p()
            _lib.call("ck_tct_create", self._descs, len(self.spec.layers), self.device,
                      params, C.byref(plan))
            self._tct_plan = plan
        return plan

    def close(self) -> None:
        for plan in getattr(self, "_tc_plans", {}).values():
            _lib.call("ck_tc_destroy", plan)
        self._tc_plans = {}
        if getattr(self, "_tct_plan", None) is not None:
            _lib.call("ck_tct_destroy", self._tct_plan)
            self._tct_plan = None
        if self._handle is not None:
            _lib.call("ck_net_destroy", self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        """The ck_net handle.  Every use may change the parameters on the
        device, so it also invalidates the tensor-core plans' weight copies."""
        if self._handle is None:
            raise StateError("network has been closed")
        self._version += 1
        return self._handle

    def set_team(self, kind: int, ctas: int, threads: int = 512) -> None:
        """Execution team of the training kernel (see ck_net_set_team)."""
        _lib.call("ck_net_set_team", self.handle, kind, ctas, threads)

    def team(self) -> tuple[int, int, int]:
        k, c, t = C.c_int(), C.c_int(), C.c_int()
        _lib.call("ck_net_get_team", self.handle, C.byref(k), C.byref(c), C.byref(t))
        return k.value, c.value, t.value

    def kernel_info(self) -> str:
        """Training kernel of this net: "specialised:<spec>" or "generic"."""
        buf = C.create_string_buffer(256)
        _lib.call("ck_net_kernel_info", self.handle, buf, len(buf))
        return buf.value.decode()

    def set_specialized(self, enable: bool) -> None:
        """Allow (default) or forbid the net's specialised training kernel."""
        _lib.call("ck_net_set_specialized", self.handle, 1 if enable else 0)

    def describe_program(self, prog: int = 0) -> str:
        """Phase program of the engine (0 train, 1 forward, 2 backward,
        3 apply, 4 eval)."""
        buf = C.create_string_buffer(1 << 14)
        _lib.call("ck_net_describe_program", self.handle, prog, buf, len(buf))
        return buf.value.decode()

    # -- parameters ----------------------------------------------------

    def _init_weights(self, seed) -> None:
        rng = np.random.default_rng(seed)
        flat = np.empty(self._n_params, dtype=np.float32)
        for _, _, shape, off in self._param_layout:
            size = int(np.prod(shape))
            flat[off:off + size] = rng.uniform(-0.05, 0.05, shape).ravel()
        self.set_flat_parameters(flat)

    def flat_parameters(self) -> np.ndarray:
        out = np.empty(self._n_params, dtype=np.float32)
        _lib.call("ck_net_get_params", self.handle, out.ctypes.data, out.size)
        return out

    def set_flat_parameters(self, flat: np.ndarray) -> None:
        flat = np.ascontiguousarray(flat, dtype=np.float32)
        if flat.size != self._n_params:
            raise DimensionError(f"expected {self._n_params} parameters, got {flat.size}")
        _lib.call("ck_net_set_params", self.handle, flat.ctypes.data, flat.size)

    def parameters(self):
        """Yield (layer_index, name, array) like the reference; arrays are
        host copies (use set_parameters / load_weights to change them)."""
        flat = self.flat_parameters()
        for idx, name, shape, off in self._param_layout:
            size = int(np.prod(shape))
            yield idx, name, flat[off:off + size].reshape(shape)

    def set_parameters(self, arrays) -> None:
        """Inverse of parameters(): iterable of (idx, name, array)."""
        flat = self.flat_parameters()
        lookup = {(i, n): (shape, off) for i, n, shape, off in self._param_layout}
        for idx, name, arr in arrays:
            shape, off = lookup[(idx, name)]
            arr = np.asarray(arr, dtype=np.float32)
            if arr.shape != shape:
                raise DimensionError(f"L{idx}_{name} has shape {arr.shape}, expected {shape}")
            flat[off:off + arr.size] = arr.ravel()
        self.set_flat_parameters(flat)

    def count_parameters(self) -> int:
        return self._n_params

    @property
    def n_classes(self) -> int:
        return self.spec.n_classes

    @property
    def input_shape(self) -> tuple[int, int, int]:
        first = self.spec.input_layer
        return first.out_maps, first.out_height, first.out_width

    # -- per-sample API ------------------------------------------------

    def _input(self, channels) -> np.ndarray:
        x = np.asarray(channels)
        if x.shape != self.input_shape:
            raise DimensionError(
                f"sample shape {x.shape} does not match input {self.input_shape}")
        return np.ascontiguousarray(x, dtype=np.float32)

    def _targets(self, targets) -> np.ndarray:
        t = np.ascontiguousarray(targets, dtype=np.float64)
        if t.shape != (self.n_classes,):
            raise DimensionError(f"targets {t.shape} do not match {self.n_classes} outputs")
        return t

    def forward(self, channels) -> np.ndarray:
        x = self._input(channels)
        y = np.empty(self.n_classes, dtype=np.float32)
        _lib.call("ck_net_forward", self.handle, x.ctypes.data, y.ctypes.data)
        return y

    def backward(self, targets) -> None:
        t = self._targets(targets)
        _lib.call("ck_net_backward", self.handle, t.ctypes.data)

    def apply_gradients(self, eta: float) -> None:
        if eta <= 0:
            raise ConfigError(f"learning rate must be > 0, got {eta}")
        _lib.call("ck_net_apply_gradients", self.handle, float(eta))

    def train_step(self, channels, targets, eta: float) -> float:
        x = self._input(channels)
        t = self._targets(targets)
        loss = C.c_double()
        _lib.call("ck_net_train_step", self.handle, x.ctypes.data, t.ctypes.data,
                  float(eta), C.byref(loss))
        return float(loss.value)

    def predict(self, channels) -> int:
        y = self.forward(channels)
        return int(np.argmax(y))

    # -- buffers -------------------------------------------------------

    def _buffer_size(self, idx, which) -> int:
        n = C.c_int64()
        _lib.call("ck_net_buffer_size", self.handle, idx, which, C.byref(n))
        return int(n.value)

    def _read_buffer(self, idx, which, dtype, shape) -> np.ndarray:
        out = np.empty(int(np.prod(shape)), dtype=dtype)
        _lib.call("ck_net_read_buffer", self.handle, idx, which, out.ctypes.data, out.size)
        return out.reshape(shape)

    # -- persistence (network.py:290-304) --------------------------------

    def save_weights(self, path) -> None:
        np.savez(path, **{f"L{idx}_{name}": arr for idx, name, arr in self.parameters()})

    def load_weights(self, path) -> None:
        with np.load(path) as data:
            arrays = []
            for idx, name, arr in self.parameters():
                key = f"L{idx}_{name}"
                if key not in data:
                    raise ConfigError(f"weight file is missing {key}")
                stored = data[key]
                if stored.shape != arr.shape:
                    raise ConfigError(f"{key} has shape {stored.shape}, expected {arr.shape}")
                arrays.append((idx, name, stored))
        self.set_parameters(arrays)
