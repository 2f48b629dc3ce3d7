"""Device runtime: layer packing, workspace management and the launches.

torch is used only as plumbing (device memory, the current CUDA stream);
every computation on the path runs in libsplitq_b200.so. There is no CPU
fallback: without a CUDA device or the native library these functions
raise.
"""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _lib
from .quantizer import QuantParams, weight_codes
from .tensor import _is_torch

_DTYPES = None


def _torch():
    import torch

    return torch


def device():
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2605_19929_b200 needs a CUDA device (sm_100a); no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _dtype_code(t):
    torch = _torch()
    return {torch.float16: _lib.F16, torch.float32: _lib.F32, torch.float64: _lib.F64,
            torch.bfloat16: _lib.BF16}[t]


def _stream():
    return C.c_void_p(_torch().cuda.current_stream().cuda_stream)


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(C.c_void_p)
    return C.c_void_p(a.data_ptr())


def _spec_struct(spec):
    if spec.bits is None or not 2 <= spec.bits <= 8:
        raise ValueError(
            f"the GPU split-linear path supports 2..8-bit integer specs (got bits={spec.bits}); "
            "identity / wide specs stay on the CPU reference")
    return _lib.QSpec(int(spec.bits), int(bool(spec.symmetric)))


def _gran(spec):
    g = spec.granularity
    return getattr(g, "value", g)


_INTS = ("d_in", "d_out", "n_main", "n_text", "n_vision", "act_bits", "act_sym", "weight_bits", "weight_sym",
         "aux_bits_floor", "use_cws", "use_mac", "r_cws", "r_mac")
_CODE_SETS = ("main", "text", "vision", "us", "vs", "uc", "vc")


def pack_arrays(layer) -> dict:
    """Everything splitq_layer_create consumes, as host numpy arrays: the
    partition, the smoothing scales and the weight side of
    forward_with_cache (layer.py:137-163) -- integer codes and fp64 column
    scales computed with the reference's own numpy expressions, so they are
    bit-exact by construction. Also the payload of a packed blob
    (layer_io.save_packed)."""
    for name in ("p_main", "p_text", "p_vision"):
        t = getattr(layer, name)
        if not getattr(t, "is_diagonal", True) or getattr(t, "scale", None) is None:
            raise ValueError("dense transforms are not supported on the GPU path")
    if _gran(layer.act_spec) != "per_token":
        raise ValueError("activation spec must be PER_TOKEN on the GPU path")
    if _gran(layer.weight_spec) == "per_token":
        raise ValueError("weight spec must be PER_CHANNEL or PER_TENSOR on the GPU path")
    p = layer.partition
    d_out = int(np.asarray(layer.w_main).shape[1])
    act, wsp = _spec_struct(layer.act_spec), _spec_struct(layer.weight_spec)
    floor = int(layer.aux_bits_floor)
    w_aux = layer.weight_spec.with_floor(floor)
    _spec_struct(w_aux)
    a = {}
    d_main = np.ascontiguousarray(layer.p_main.scale, dtype=np.float64)
    a["scale_main"] = d_main
    a["scale_text"] = (np.ascontiguousarray(layer.p_text.scale, dtype=np.float64) if len(p.c_text)
                       else np.zeros(0))
    a["scale_vision"] = (np.ascontiguousarray(layer.p_vision.scale, dtype=np.float64) if len(p.c_vision)
                         else np.zeros(0))
    for k in ("c_main", "c_text", "c_vision"):
        a[k] = np.ascontiguousarray(getattr(p, k), dtype=np.int64)
    w_prime = np.asarray(layer.w_main, np.float64) / d_main[:, np.newaxis]  # apply_inv_left
    ints = dict(d_in=int(p.dim), d_out=d_out, n_main=len(p.c_main), n_text=len(p.c_text),
                n_vision=len(p.c_vision), act_bits=act.bits, act_sym=act.symmetric, weight_bits=wsp.bits,
                weight_sym=wsp.symmetric, aux_bits_floor=floor, use_cws=int(bool(layer.use_cws)),
                use_mac=int(bool(layer.use_mac)), r_cws=0, r_mac=0)

    def put(name, m, spec):
        q, s = weight_codes(m, spec)
        a["q_" + name] = np.ascontiguousarray(q, dtype=np.int8)
        a["s_" + name] = np.ascontiguousarray(s, dtype=np.float64)

    if layer.use_cws:
        br = layer.branch_smooth
        v_eff = br.effective_v()
        r_pre = w_prime - br.u_star @ v_eff  # layer.py:144 (same numpy/BLAS call)
        put("main", r_pre, layer.weight_spec)
        put("us", br.u_star, w_aux)
        put("vs", v_eff, w_aux)
        ints["r_cws"] = int(br.rank)
    else:
        put("main", w_prime, layer.weight_spec)
    if layer.use_mac:
        br = layer.branch_comp
        put("uc", br.u_star, w_aux)
        put("vc", br.effective_v(), w_aux)
        ints["r_mac"] = int(br.rank)
    if len(p.c_text):
        put("text", np.asarray(layer.w_text, np.float64) / a["scale_text"][:, np.newaxis], w_aux)
    if len(p.c_vision):
        put("vision", np.asarray(layer.w_vision, np.float64) / a["scale_vision"][:, np.newaxis], w_aux)
    for k, v in ints.items():
        a[k] = np.array(v, dtype=np.int64)
    return a


class GpuLayer:
    """A SplitLayer packed on one device: the C handle plus its geometry.
    Built from a layer (weight codes computed here) or from the arrays of a
    packed blob (layer_io.load_packed: no recomputation)."""

    def __init__(self, layer=None, dev=None, arrays=None):
        lib = _lib.load()
        dev = dev or device()
        a = pack_arrays(layer) if arrays is None else arrays
        keep = []

        def arr(name, dt):
            if name not in a:
                return None
            v = np.ascontiguousarray(a[name], dtype=dt)
            keep.append(v)
            return _ptr(v)

        iv = {k: int(a[k]) for k in _INTS}
        desc = _lib.LayerDesc()
        desc.d_in, desc.d_out = iv["d_in"], iv["d_out"]
        desc.n_main, desc.n_text, desc.n_vision = iv["n_main"], iv["n_text"], iv["n_vision"]
        desc.c_main, desc.c_text, desc.c_vision = (arr("c_main", np.int64), arr("c_text", np.int64),
                                                   arr("c_vision", np.int64))
        desc.scale_main, desc.scale_text, desc.scale_vision = (arr("scale_main", np.float64),
                                                               arr("scale_text", np.float64),
                                                               arr("scale_vision", np.float64))
        desc.act = _lib.QSpec(iv["act_bits"], iv["act_sym"])
        desc.weight = _lib.QSpec(iv["weight_bits"], iv["weight_sym"])
        desc.aux_bits_floor = iv["aux_bits_floor"]
        desc.use_cws, desc.use_mac = iv["use_cws"], iv["use_mac"]
        desc.r_cws, desc.r_mac = iv["r_cws"], iv["r_mac"]
        for name in _CODE_SETS:
            setattr(desc, "q_" + name, arr("q_" + name, np.int8))
            setattr(desc, "s_" + name, arr("s_" + name, np.float64))
        handle = C.c_void_p()
        _lib.check(lib.splitq_layer_create(C.byref(desc), int(dev.index or 0), C.byref(handle)))
        self.handle = handle
        self.device = dev
        self.d_in, self.d_out = iv["d_in"], iv["d_out"]
        self._ws = {}
        self._finalizer = weakref.finalize(self, lib.splitq_layer_destroy, handle)

    def layout(self, tokens: int) -> _lib.WsLayout:
        lay = _lib.WsLayout()
        _lib.check(_lib.load().splitq_workspace_layout(self.handle, int(tokens), C.byref(lay)))
        return lay

    def workspace(self, tokens: int):
        torch = _torch()
        ws = self._ws.get(tokens)
        if ws is None:
            lay = self.layout(tokens)
            ws = torch.empty(int(lay.total_bytes), dtype=torch.uint8, device=self.device)
            self._ws = {tokens: ws}  # keep the latest size only
        return ws

    def run(self, x, tags, y=None, out_dtype=None, raw=False, check=True, ws=None,
            profile=False, unpacked=False):
        """Launch the forward on the current stream. x: CUDA [T x >=d_in]
        (f16/bf16/f32/f64, unit column stride), tags: CUDA uint8 [T].
        Without ws the layer's cached workspace is used: calls that may run
        concurrently (other streams or threads) must each pass their own."""
        torch = _torch()
        lib = _lib.load()
        if not (_is_torch(x) and _is_torch(tags)):
            raise ValueError("run() takes CUDA tensors (use forward() for host arrays)")
        if x.ndim != 2:
            raise ValueError(f"matrix must be 2-D, got ndim={x.ndim}")
        T = int(x.shape[0])
        if x.shape[1] != self.d_in:
            raise ValueError("batch width does not match partition dim")
        if x.device != self.device or tags.device != self.device:
            raise ValueError(f"x and tags must be on {self.device}")
        if x.dtype not in (torch.float16, torch.bfloat16, torch.float32, torch.float64):
            raise ValueError(f"unsupported activation dtype {x.dtype}")
        if x.stride(1) != 1:
            x = x.contiguous()
        tags = tags.reshape(-1).to(torch.uint8).contiguous()
        if tags.numel() != T:
            raise ValueError("tags length must match the number of rows")
        if ws is None:
            ws = self.workspace(T)
        if raw:
            y = torch.empty((2, T, self.d_out), dtype=torch.int32, device=self.device)
            ydt = _lib.F32
        else:
            out_dtype = out_dtype or torch.float32
            if y is None:
                y = torch.empty((T, self.d_out), dtype=out_dtype, device=self.device)
            if (not _is_torch(y) or y.device != self.device or y.ndim != 2
                    or tuple(y.shape) != (T, self.d_out) or y.stride(-1) != 1
                    or y.dtype not in (torch.float32, torch.float16, torch.bfloat16)):
                raise ValueError(f"y must be a CUDA f32/f16/bf16 [{T} x {self.d_out}] tensor with unit "
                                 f"column stride on {self.device}")
            ydt = _dtype_code(y.dtype)
        y_ld = y.stride(-2)
        _lib.check(lib.splitq_forward(self.handle, _ptr(x), _dtype_code(x.dtype), x.stride(0),
                                      _ptr(tags), T, _ptr(y), ydt, y_ld, _ptr(ws),
                                      ws.numel(), _stream(),
                                      (_lib.FWD_RAW if raw else 0) | (_lib.FWD_PROFILE if profile else 0)
                                      | (_lib.FWD_UNPACKED if unpacked else 0)))
        if check:
            st = C.c_int32()
            _lib.check(lib.splitq_read_status(_ptr(ws), _stream(), C.byref(st)))
        return y


    def profile_read(self):
        """Summed stage times (ms) of the profiled calls since the last read:
        (quantize, low-rank first stages, split GEMM), number of calls."""
        ms = (C.c_double * 3)()
        calls = C.c_int32()
        _lib.check(_lib.load().splitq_profile_read(self.handle, ms, C.byref(calls)))
        return list(ms), calls.value


_PACKED: dict = {}


def _fingerprint(layer) -> bytes:
    """Cheap content key of a layer: shapes, specs, the partition, the
    smoothing scales, the branch gates and a strided sample of every weight
    matrix. A layer whose arrays are edited in place after its first forward
    (outside those samples) must be re-packed explicitly (GpuLayer(layer))."""
    import hashlib

    h = hashlib.blake2b(digest_size=16)
    h.update(repr((layer.act_spec, layer.weight_spec, getattr(layer, "aux_bits_floor", None),
                   bool(layer.use_cws), bool(layer.use_mac))).encode())

    def put(a, sample=False):
        if a is None:
            h.update(b"-")
            return
        a = np.asarray(a)
        h.update(repr((a.shape, a.dtype.str)).encode())
        flat = a.reshape(-1)
        if sample and flat.size > 65536:
            flat = flat[:: flat.size // 65536 + 1]
        h.update(np.ascontiguousarray(flat).tobytes())

    p = layer.partition
    for c in (p.c_main, p.c_text, p.c_vision):
        put(c)
    for t in (layer.p_main, layer.p_text, layer.p_vision):
        put(getattr(t, "scale", None))
    for w in (layer.w_main, layer.w_text, layer.w_vision):
        put(w, sample=True)
    for br in (getattr(layer, "branch_smooth", None), getattr(layer, "branch_comp", None)):
        if br is not None:
            put(br.gate)
            put(br.u_star, sample=True)
            put(br.v_base, sample=True)
    return h.digest()


def packed(layer) -> GpuLayer:
    """Pack a layer once per (object, device, content fingerprint). Objects
    without weakref support are not cached (their id may be reused)."""
    if isinstance(layer, GpuLayer):
        return layer
    dev = device()
    try:
        weakref.ref(layer)
    except TypeError:
        return GpuLayer(layer, dev)
    key = (id(layer), dev.index)
    fp = _fingerprint(layer)
    hit = _PACKED.get(key)
    if hit is not None and hit[0] == fp:
        return hit[1]
    g = GpuLayer(layer, dev)
    if hit is None:
        weakref.finalize(layer, _PACKED.pop, key, None)
    _PACKED[key] = (fp, g)
    return g


def forward(layer, batch, out_dtype=None):
    torch = _torch()
    g = packed(layer)
    dev = g.device
    data, tags = batch.data, batch.tags
    if _is_torch(data):
        x = data.to(dev)
        t = tags.to(dev) if _is_torch(tags) else torch.as_tensor(np.asarray(tags, np.uint8), device=dev)
        return g.run(x, t, out_dtype=out_dtype)
    x = torch.from_numpy(np.ascontiguousarray(data, dtype=np.float64)).to(dev)
    t = torch.from_numpy(np.ascontiguousarray(tags, dtype=np.uint8)).to(dev)
    y = g.run(x, t, out_dtype=torch.float32)
    return y.cpu().numpy().astype(np.float64)


def quantize_rows(x, spec):
    """PER_TOKEN quantization on the GPU -> (codes q int64 ndarray, QuantParams)."""
    torch = _torch()
    lib = _lib.load()
    dev = device()
    host = not _is_torch(x)
    if host:
        xa = np.asarray(x, dtype=np.float64)
        if xa.ndim != 2:
            raise ValueError(f"matrix must be 2-D, got ndim={xa.ndim}")
        xt = torch.from_numpy(np.ascontiguousarray(xa)).to(dev)
    else:
        xt = x.to(dev)
        if xt.ndim != 2:
            raise ValueError(f"matrix must be 2-D, got ndim={xt.ndim}")
        if xt.stride(1) != 1:
            xt = xt.contiguous()
    rows, cols = int(xt.shape[0]), int(xt.shape[1])
    if rows == 0 or cols == 0:
        return np.zeros((rows, cols), np.int64), QuantParams(np.ones(rows), np.zeros(rows, np.int64))
    ld = (cols + 15) // 16 * 16
    codes = torch.empty((rows, ld), dtype=torch.int8, device=dev)
    scales = torch.empty(rows, dtype=torch.float64, device=dev)
    zps = torch.empty(rows, dtype=torch.int32, device=dev)
    status = torch.zeros(4, dtype=torch.int32, device=dev)
    centered = C.c_int32()
    _lib.check(lib.splitq_quantize_rows(_ptr(xt), _dtype_code(xt.dtype), xt.stride(0), rows, cols,
                                        _spec_struct(spec), _ptr(codes), ld, _ptr(scales),
                                        _ptr(zps), _ptr(status), C.byref(centered), _stream()))
    st = C.c_int32()
    _lib.check(lib.splitq_read_status(_ptr(status), _stream(), C.byref(st)))
    s = scales.cpu().numpy()
    z = zps.cpu().numpy().astype(np.int64)
    c = codes[:, :cols].cpu().numpy().astype(np.int64)
    q = c + z[:, None] if centered.value else (c & 0xFF)
    return q, QuantParams(s, z)
