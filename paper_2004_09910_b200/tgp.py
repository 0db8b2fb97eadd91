"""Thin ctypes binding of the tgp C ABI (include/tgp.h).  Argument marshalling only: every step of
the hot path runs in libtgp.so's CUDA kernels.  There is no fallback: if the library is missing or
a call fails, a TgpError is raised.

Tensors passed to the device calls are torch CUDA tensors (PyTorch is used for device memory and
streams only); parameters are exchanged as numpy float32 arrays on the host.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TGP_LIB") or os.path.join(_HERE, "libtgp.so")

KIND = {"linear": 0, "resmlp": 1, "merge": 2, "batchnorm": 3, "embed": 4, "transformer": 5, "lmhead": 6,
        "layernorm": 7, "dropout": 8}
ACT = {"none": 0, "relu": 1, "gelu": 2}
CKPT = {"always": 0, "except_last": 1, "never": 2}
DTYPE = {"fp32": 0, "bf16": 1}
# schedule record kinds (tgp_schedule)
F, RECOMPUTE, B, COPY_F, COPY_B, SKIP_F, SKIP_B, W = range(8)


class TgpError(RuntimeError):
    """A tgp_* call returned a status != 0 (`rc`, include/tgp.h tgp_status)."""

    def __init__(self, msg, rc=None):
        super().__init__(msg)
        self.rc = rc


class Layer(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("d_in", ctypes.c_int32), ("d_out", ctypes.c_int32),
                ("d_hidden", ctypes.c_int32), ("act", ctypes.c_int32), ("dropout", ctypes.c_float),
                ("stash_route", ctypes.c_int32), ("pop_route", ctypes.c_int32), ("n_heads", ctypes.c_int32),
                ("seq", ctypes.c_int32), ("vocab", ctypes.c_int32)]


_lib = None
_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64

_SIGS = {
    "tgp_balance": [ctypes.POINTER(ctypes.c_double), _I32, _I32, ctypes.POINTER(_I32)],
    "tgp_profile_size": [_P, _I32, _I32, ctypes.POINTER(ctypes.c_double)],
    "tgp_split": [_I32, _I32, ctypes.POINTER(_I32)],
    "tgp_schedule": [_I32, _I32, _I32, ctypes.POINTER(_I32), _I32, ctypes.POINTER(_I32), _I64,
                     ctypes.POINTER(_I64)],
    "tgp_schedule_ablation": [_I32, _I32, _I32, ctypes.POINTER(_I32), _I32, _I32, ctypes.c_uint64,
                              ctypes.POINTER(_I32), _I64, ctypes.POINTER(_I64)],
    "tgp_copy_stats": [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64)],
    "tgp_create": [ctypes.POINTER(Layer), _I32, ctypes.POINTER(_I32), _I32, _I32, _I32, ctypes.POINTER(_I32),
                   _I32, _I32, ctypes.c_uint64, ctypes.POINTER(_P)],
    "tgp_destroy": [_P],
    "tgp_ipc_export": [_P, _I32, _P, _I64, ctypes.POINTER(_I64)],
    "tgp_ipc_import": [_P, _I32, _P, _I64],
    "tgp_connect": [_P],
    "tgp_forward": [_P, _P, _I32, _P],
    "tgp_mse_loss_grad": [_P, _P, _P, _I32, _P, ctypes.POINTER(ctypes.c_double)],
    "tgp_ce_loss_grad": [_P, _P, _P, _I32, _P, ctypes.POINTER(ctypes.c_double)],
    "tgp_backward": [_P, _P, _P],
    "tgp_step": [_P, ctypes.c_float],
    "tgp_backward_step": [_P, _P, _P, ctypes.c_float],
    "tgp_forward_async": [_P, _P, _I32, _P, _P],
    "tgp_mse_loss_grad_async": [_P, _P, _P, _I32, _P, _P, _P],
    "tgp_backward_async": [_P, _P, _P, _P],
    "tgp_backward_step_async": [_P, _P, _P, ctypes.c_float, _P],
    "tgp_step_async": [_P, ctypes.c_float, _P],
    "tgp_sync": [_P],
    "tgp_num_params": [_P, ctypes.POINTER(_I32)],
    "tgp_param_info": [_P, _I32, ctypes.POINTER(_I32), ctypes.POINTER(_I32), ctypes.POINTER(_I64)],
    "tgp_set_param": [_P, _I32, _P],
    "tgp_get_param": [_P, _I32, _P],
    "tgp_get_grad": [_P, _I32, _P],
    "tgp_init_params": [_P, ctypes.c_uint64],
    "tgp_get_bn_running": [_P, _I32, _P, _P],
    "tgp_get_issue_log": [_P, ctypes.POINTER(_I32), _I64, ctypes.POINTER(_I64)],
    "tgp_set_trace": [_P, _I32],
    "tgp_get_timeline": [_P, ctypes.POINTER(_I64), _I64, ctypes.POINTER(_I64)],
    "tgp_kernel_count": [_P, ctypes.POINTER(_I64)],
    "tgp_set_option": [_P, ctypes.c_char_p, _I64],
    "tgp_last_error": [],
    "tgp_bench_dominant_gemm": [_P, _I32, _I32, _I32, ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I64)],
    "tgp_debug_stream_read": [_P, _I32, _P, _I64, ctypes.POINTER(_I64)],
    "tgp_stream_enabled": [_P, _I32, ctypes.POINTER(_I32)],
    "tgp_profile_layers": [_P, _I32, _I32, _I32, ctypes.POINTER(ctypes.c_double)],
    "tgp_memory": [_P, _I32, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I64)],
    "tgp_memory_breakdown": [_P, _I32, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I32)],
    "tgp_test_gemm_bf16": [_P, _P, _P, _I32, _I32, _I32, _I32, _I32, _I32, _P],
    "tgp_bench_transport": [_I32, _I32, _I64, _I32, _I32, ctypes.POINTER(ctypes.c_double),
                            ctypes.POINTER(ctypes.c_double)],
}


def lib():
    """Load libtgp.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise TgpError(f"{LIB_PATH} not found: build it with `python -m paper_2004_09910_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_char_p if name == "tgp_last_error" else (None if name == "tgp_destroy" else ctypes.c_int)
        _lib = L
    return _lib


def exported_symbols():
    return sorted(_SIGS)


def _check(rc, what):
    if rc != 0:
        msg = lib().tgp_last_error()
        raise TgpError(f"{what} failed ({rc}): {msg.decode() if msg else ''}", rc)


def _ptr(t):
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return ctypes.c_void_p(t.data_ptr())
    return ctypes.c_void_p(int(t))


def _ready(*tensors):
    """The library works on its own non-blocking streams: make sure the work torch queued on the
    caller's current stream for these tensors (their producers) has finished before handing them over."""
    import torch

    devs = {t.device for t in tensors if t is not None and hasattr(t, "device") and t.device.type == "cuda"}
    for d in devs:
        torch.cuda.current_stream(d).synchronize()


# ------------------------------------------------------------------ pure host helpers
def balance(costs, n):
    c = (ctypes.c_double * len(costs))(*[float(v) for v in costs])
    out = (_I32 * n)()
    _check(lib().tgp_balance(c, len(costs), n, out), "tgp_balance")
    return list(out)


def profile_size(layers, rows):
    """Per-layer bytes (tgp_profile_size): 8 x parameters + rows x d_out x 4 (§4.2.2)."""
    arr = to_c_layers(layers)
    out = (ctypes.c_double * len(layers))()
    _check(lib().tgp_profile_size(arr, len(layers), rows, out), "tgp_profile_size")
    return list(out)


def balance_by_size(layers, n_parts, rows):
    """Size-based partition (SPEC profile_size + blockpartition): min-max contiguous blocks of the
    per-layer bytes.  Returns (balance, bytes)."""
    sizes = profile_size(layers, rows)
    return balance(sizes, n_parts), sizes


def split(B, m):
    out = (_I32 * m)()
    _check(lib().tgp_split(B, m, out), "tgp_split")
    return list(out)


def schedule(m, n, checkpoint="except_last", routes=(), relay=False, order_seed=0):
    """tgp_schedule records [n_rec][8]; relay / order_seed select the Table 1 ablation variants
    (tgp_schedule_ablation)."""
    routes = list(routes)
    r = (_I32 * max(1, 2 * len(routes)))(*[v for pr in routes for v in pr])
    cnt = _I64()
    if relay or order_seed:
        call = lambda buf, cap: lib().tgp_schedule_ablation(m, n, CKPT[checkpoint], r, len(routes), int(bool(relay)),
                                                             order_seed, buf, cap, ctypes.byref(cnt))
    else:
        call = lambda buf, cap: lib().tgp_schedule(m, n, CKPT[checkpoint], r, len(routes), buf, cap, ctypes.byref(cnt))
    _check(call(None, 0), "tgp_schedule")
    buf = (_I32 * (8 * cnt.value))()
    _check(call(buf, cnt.value), "tgp_schedule")
    return np.frombuffer(buf, dtype=np.int32).reshape(-1, 8).copy()


def test_gemm_bf16(A, Bm, D, M, N, K, a_mn, b_mn, splits=0, stream=None):
    _ready(A, Bm, D)
    _check(lib().tgp_test_gemm_bf16(_ptr(A), _ptr(Bm), _ptr(D), M, N, K, int(a_mn), int(b_mn), splits,
                                    _ptr(stream) if stream is not None else None), "tgp_test_gemm_bf16")


def to_c_layers(layers):
    arr = (Layer * len(layers))()
    for q, L in enumerate(layers):
        arr[q] = Layer(KIND[L["kind"]], L["d_in"], L["d_out"], L.get("d_hidden", 0), ACT[L.get("act", "none")],
                       float(L.get("dropout", 0.0)), L.get("stash", -1), L.get("pop", -1), L.get("n_heads", 0),
                       L.get("seq", 0), L.get("vocab", 0))
    return arr


class Pipeline:
    """A GPipe pipeline over this process's local partitions (tgp_ctx)."""

    def __init__(self, layers, *, chunks, devices, balance=None, checkpoint="except_last", max_batch,
                 dtype="bf16", seed=0):
        self.layers = layers
        self.n = len(devices)
        self.m = chunks
        self.devices = list(devices)
        self._c_layers = to_c_layers(layers)
        bal = None if balance is None else (_I32 * self.n)(*balance)
        dev = (_I32 * self.n)(*devices)
        h = _P()
        _check(lib().tgp_create(self._c_layers, len(layers), bal, self.n, chunks, CKPT[checkpoint], dev, max_batch,
                                DTYPE[dtype], seed, ctypes.byref(h)), "tgp_create")
        self.h = h
        n = _I32()
        _check(lib().tgp_num_params(self.h, ctypes.byref(n)), "tgp_num_params")
        self.n_params = n.value

    def close(self):
        if self.h:
            lib().tgp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- multi-process wiring
    def ipc_export(self, part):
        n = _I64()
        _check(lib().tgp_ipc_export(self.h, part, None, 0, ctypes.byref(n)), "tgp_ipc_export")
        buf = ctypes.create_string_buffer(n.value)
        _check(lib().tgp_ipc_export(self.h, part, buf, n.value, ctypes.byref(n)), "tgp_ipc_export")
        return buf.raw

    def ipc_import(self, part, blob):
        buf = ctypes.create_string_buffer(blob, len(blob))
        _check(lib().tgp_ipc_import(self.h, part, buf, len(blob)), "tgp_ipc_import")

    def connect(self):
        _check(lib().tgp_connect(self.h), "tgp_connect")

    # ---- training step
    def forward(self, x, B, y):
        _ready(x, y)
        _check(lib().tgp_forward(self.h, _ptr(x), B, _ptr(y)), "tgp_forward")

    def mse_loss_grad(self, y, t, B, dy):
        loss = ctypes.c_double()
        _ready(y, t, dy)
        _check(lib().tgp_mse_loss_grad(self.h, _ptr(y), _ptr(t), B, _ptr(dy), ctypes.byref(loss)),
               "tgp_mse_loss_grad")
        return loss.value

    def ce_loss_grad(self, y, t, B, dy):
        """Token cross-entropy (C5): y, dy [B, vocab] fp32, t [B] int32 on the last partition's device."""
        loss = ctypes.c_double()
        _ready(y, t, dy)
        _check(lib().tgp_ce_loss_grad(self.h, _ptr(y), _ptr(t), B, _ptr(dy), ctypes.byref(loss)),
               "tgp_ce_loss_grad")
        return loss.value

    def backward(self, dy, dx=None):
        _ready(dy, dx)
        _check(lib().tgp_backward(self.h, _ptr(dy), _ptr(dx)), "tgp_backward")

    def step(self, lr):
        _check(lib().tgp_step(self.h, ctypes.c_float(lr)), "tgp_step")

    def backward_step(self, dy, lr, dx=None):
        """tgp_backward + tgp_step(lr) with SGD fused into W_j (fused weight gradients not stored)."""
        _ready(dy, dx)
        _check(lib().tgp_backward_step(self.h, _ptr(dy), _ptr(dx), ctypes.c_float(lr)), "tgp_backward_step")

    # ---- asynchronous, stream-ordered variants (include/tgp.h): no host wait, no _ready(); the
    # work is ordered after what is queued on `stream` (default: torch's current stream of the
    # tensor's device) and `stream` waits for it
    @staticmethod
    def _stream(stream, t):
        if stream is not None:
            return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
        import torch

        return ctypes.c_void_p(torch.cuda.current_stream(t.device if t is not None else None).cuda_stream)

    def forward_async(self, x, B, y, stream=None):
        _check(lib().tgp_forward_async(self.h, _ptr(x), B, _ptr(y), self._stream(stream, x if x is not None else y)),
               "tgp_forward_async")

    def mse_loss_grad_async(self, y, t, B, dy, loss_dev=None, stream=None):
        """loss_dev: a float64 CUDA tensor of >= 1 element on y's device (or None)."""
        _check(lib().tgp_mse_loss_grad_async(self.h, _ptr(y), _ptr(t), B, _ptr(dy), _ptr(loss_dev),
                                             self._stream(stream, y)), "tgp_mse_loss_grad_async")

    def backward_async(self, dy, dx=None, stream=None):
        _check(lib().tgp_backward_async(self.h, _ptr(dy), _ptr(dx), self._stream(stream, dy if dy is not None else dx)),
               "tgp_backward_async")

    def backward_step_async(self, dy, lr, dx=None, stream=None):
        _check(lib().tgp_backward_step_async(self.h, _ptr(dy), _ptr(dx), ctypes.c_float(lr),
                                             self._stream(stream, dy if dy is not None else dx)),
               "tgp_backward_step_async")

    def step_async(self, lr, stream=None):
        _check(lib().tgp_step_async(self.h, ctypes.c_float(lr), self._stream(stream, None)), "tgp_step_async")

    def sync(self):
        _check(lib().tgp_sync(self.h), "tgp_sync")

    # ---- parameters
    def param_info(self, idx):
        layer, part, numel = _I32(), _I32(), _I64()
        _check(lib().tgp_param_info(self.h, idx, ctypes.byref(layer), ctypes.byref(part), ctypes.byref(numel)),
               "tgp_param_info")
        return layer.value, part.value, numel.value

    def set_param(self, idx, arr):
        a = np.ascontiguousarray(arr, dtype=np.float32)
        _check(lib().tgp_set_param(self.h, idx, a.ctypes.data_as(_P)), "tgp_set_param")

    def get_param(self, idx, shape=None):
        _, _, numel = self.param_info(idx)
        a = np.empty(numel, dtype=np.float32)
        _check(lib().tgp_get_param(self.h, idx, a.ctypes.data_as(_P)), "tgp_get_param")
        return a.reshape(shape) if shape is not None else a

    def get_grad(self, idx, shape=None):
        _, _, numel = self.param_info(idx)
        a = np.empty(numel, dtype=np.float32)
        _check(lib().tgp_get_grad(self.h, idx, a.ctypes.data_as(_P)), "tgp_get_grad")
        return a.reshape(shape) if shape is not None else a

    def init_params(self, seed=0):
        _check(lib().tgp_init_params(self.h, seed), "tgp_init_params")

    def bn_running(self, layer, d):
        mean = np.empty(d, np.float32)
        var = np.empty(d, np.float32)
        _check(lib().tgp_get_bn_running(self.h, layer, mean.ctypes.data_as(_P), var.ctypes.data_as(_P)),
               "tgp_get_bn_running")
        return mean, var

    # ---- introspection
    def issue_log(self):
        n = _I64()
        _check(lib().tgp_get_issue_log(self.h, None, 0, ctypes.byref(n)), "tgp_get_issue_log")
        buf = (_I32 * (8 * max(1, n.value)))()
        _check(lib().tgp_get_issue_log(self.h, buf, n.value, ctypes.byref(n)), "tgp_get_issue_log")
        return np.frombuffer(buf, dtype=np.int32)[: 8 * n.value].reshape(-1, 8).copy()

    def set_trace(self, on=True):
        _check(lib().tgp_set_trace(self.h, int(on)), "tgp_set_trace")

    def timeline(self):
        n = _I64()
        _check(lib().tgp_get_timeline(self.h, None, 0, ctypes.byref(n)), "tgp_get_timeline")
        buf = (_I64 * (6 * max(1, n.value)))()
        _check(lib().tgp_get_timeline(self.h, buf, n.value, ctypes.byref(n)), "tgp_get_timeline")
        return np.frombuffer(buf, dtype=np.int64)[: 6 * n.value].reshape(-1, 6).copy()

    def kernel_count(self):
        n = _I64()
        _check(lib().tgp_kernel_count(self.h, ctypes.byref(n)), "tgp_kernel_count")
        return n.value

    def bench_dominant_gemm(self, part, B, reps=3):
        ms, by, n = ctypes.c_double(), ctypes.c_double(), _I64()
        _check(lib().tgp_bench_dominant_gemm(self.h, part, B, reps, ctypes.byref(ms), ctypes.byref(by),
                                             ctypes.byref(n)), "tgp_bench_dominant_gemm")
        return ms.value, by.value, n.value

    def profile_layers(self, part, B, reps=5):
        """Per-layer forward + backward device time (ms) of local partition `part` (tgp_profile_layers)."""
        n = len({self.param_info(i)[0] for i in range(self.n_params) if self.param_info(i)[1] == part})
        out = (ctypes.c_double * max(1, n))()
        _check(lib().tgp_profile_layers(self.h, part, B, reps, out), "tgp_profile_layers")
        return [out[k] for k in range(n)]

    def memory(self, part):
        """Static memory plan of local partition `part`: dict(used, reserved, params) in bytes."""
        u, r, p = _I64(), _I64(), _I64()
        _check(lib().tgp_memory(self.h, part, ctypes.byref(u), ctypes.byref(r), ctypes.byref(p)), "tgp_memory")
        return {"used": u.value, "reserved": r.value, "params": p.value}

    def memory_breakdown(self, part):
        """What checkpointing changes (tgp_memory_breakdown): dict(stash, slots, n_slots) -- the bf16
        dW-operand / skip stash (whole mini-batch, every mode) and the per-slot fp32 activations."""
        st, sl, ns = _I64(), _I64(), _I32()
        _check(lib().tgp_memory_breakdown(self.h, part, ctypes.byref(st), ctypes.byref(sl), ctypes.byref(ns)),
               "tgp_memory_breakdown")
        return {"stash": st.value, "slots": sl.value, "n_slots": ns.value}

    def copy_stats(self):
        """(payload bytes, messages) pushed by this process since creation (tgp_copy_stats)."""
        b, n = _I64(), _I64()
        _check(lib().tgp_copy_stats(self.h, ctypes.byref(b), ctypes.byref(n)), "tgp_copy_stats")
        return b.value, n.value

    def stream_enabled(self, part):
        on = _I32()
        _check(lib().tgp_stream_enabled(self.h, part, ctypes.byref(on)), "tgp_stream_enabled")
        return bool(on.value)

    def set_option(self, name, value):
        _check(lib().tgp_set_option(self.h, name.encode(), int(value)), "tgp_set_option")


def bench_transport(dev_src, dev_dst, nbytes, mode=0, reps=50):
    """Per-message device time of the stage-boundary transport (tgp_bench_transport): mode 0 = SM push
    kernel + release flag, 1 = copy engine + stream-written flag.  Returns (us_stream, us_pingpong)."""
    a, b = ctypes.c_double(), ctypes.c_double()
    _check(lib().tgp_bench_transport(dev_src, dev_dst, int(nbytes), mode, reps, ctypes.byref(a), ctypes.byref(b)),
           "tgp_bench_transport")
    return a.value, b.value


def balance_by_time(layers, n_parts, *, batch, chunks, device=0, dtype="bf16", reps=5, seed=0):
    """Profile-based partition ("resource consumption is computed by profiling"):
    time every layer's forward + backward on one device (tgp_profile_layers, one micro-batch of
    batch / chunks rows), then the min-max contiguous partition of those costs (tgp_balance).
    Returns (balance, costs_ms)."""
    P = Pipeline(layers, chunks=chunks, devices=[device], balance=[len(layers)], checkpoint="never",
                 max_batch=batch, dtype=dtype, seed=seed)
    try:
        P.init_params(seed)
        costs = P.profile_layers(0, batch, reps)
    finally:
        P.close()
    return balance(costs, n_parts), costs
