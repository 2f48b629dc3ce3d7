"""Calibration caller of the path on the GPU (reference:
pkg/src/modquant/layer.py:100-172 forward_with_cache, calibrate.py:128-270).

``forward_with_cache`` returns the forward output and every intermediate the
straight-through (STE) gradient needs, in fp64 on the device:

  * quantization (compute_params + fake_quantize, quantizer.py:104-155) runs
    through the K1 kernel (``torch.ops.splitq.quantize_per_token`` over the
    fp64 rows; PER_CHANNEL groups are the rows of the transposed matrix), so
    codes, scales and zero points are bit-identical to the reference's and
    the fake-quantized values (q - z) S are the reference's fp64 values;
  * the clamp masks (quantizer.py:158-167) come from the same exact scales:
    1 where rha(m / S) + z is inside [q_min, q_max];
  * the fp64 matmuls are cuBLAS DGEMMs (library GEMMs: the result differs
    from the reference's OpenBLAS only by summation order).

``analytic_gradient`` and ``calibrate`` are the reference's STE gradient and
cosine-decayed gradient descent with the device cache; the host keeps only
the flat parameter vector (log-scales and gates, a few thousand values).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import transform as tr
from .tensor import _is_torch

MAX_FD_PARAMS = 4096
_LOG_LO = np.log(tr.DIAG_EPS)
_LOG_HI = np.log(tr.DIAG_MAX)


def _torch():
    import torch

    return torch


@dataclass(frozen=True)
class CalibConfig:  # calibrate.py:27-47
    steps: int = 200
    learning_rate: float = 1.0
    seed: int = 0
    learn_p_main: bool = True
    learn_p_text: bool = True
    learn_p_vision: bool = True
    learn_gates: bool = True
    grad_mode: str = "analytic"  # or "fd"
    fd_step: float = 1e-4

    def __post_init__(self):
        if self.learning_rate <= 0:
            raise ValueError("learning_rate must be positive")
        if self.steps < 1:
            raise ValueError("steps must be positive")
        if self.grad_mode not in ("analytic", "fd"):
            raise ValueError(f"unknown grad_mode {self.grad_mode!r}")


@dataclass
class LossTrace:  # calibrate.py:50-60
    losses: list[float] = field(default_factory=list)

    @property
    def best_loss(self) -> float:
        return min(self.losses)

    @property
    def best_step(self) -> int:
        return int(np.argmin(self.losses))


class NonFiniteLossError(RuntimeError):  # calibrate.py:63-66
    def __init__(self, step: int):
        super().__init__(f"non-finite loss at step {step}")
        self.step = step


# ------------------------------------------------------------------ device tensors

class _Dev:
    """Host arrays uploaded once per calibration run (weights and branch
    factors are fixed; only transforms and gates change between steps)."""

    def __init__(self):
        import torch

        from .runtime import device

        self.dev = device()
        self.torch = torch
        self._keep = {}

    def __call__(self, a):
        torch = self.torch
        if _is_torch(a):
            return a.to(self.dev, torch.float64)
        a = np.asarray(a)
        hit = self._keep.get(id(a))
        if hit is not None and hit[0] is a:
            return hit[1]
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(self.dev)
        self._keep[id(a)] = (a, t)
        return t


def _quantized(m, spec):
    """(fake-quantized value, STE mask) of an fp64 device matrix with fresh
    params (layer.py:100-103). PER_TOKEN groups are rows, PER_CHANNEL groups
    columns (the rows of m^T), PER_TENSOR one group."""
    torch = _torch()
    from . import ops  # noqa: F401  (registers torch.ops.splitq)

    if spec.is_identity:
        return m.clone(), torch.ones_like(m)
    g = getattr(spec.granularity, "value", spec.granularity)
    rows, cols = m.shape
    if rows == 0 or cols == 0:
        return m.clone(), torch.ones_like(m)
    src = m if g == "per_token" else (m.t() if g == "per_channel" else m.reshape(1, -1))
    src = src.contiguous()
    codes, s, z, st = torch.ops.splitq.quantize_per_token(src, int(spec.bits), bool(spec.symmetric))
    if int(st[0].item()):
        from .ops import check_status

        check_status(st)
    n = src.shape[1]
    c = codes[:, :n].to(torch.int64)
    zf = z.to(torch.float64)[:, None]
    centered = bool(spec.symmetric) or spec.bits <= 7
    q = (c.to(torch.float64) + zf) if centered else (c & 0xFF).to(torch.float64)
    sf = s[:, None]
    fq = (q - zf) * sf  # fake_quantize (quantizer.py:154-155)
    v = src / sf  # clamp_mask (quantizer.py:158-167): rha(m / S) + z in range
    qr = torch.sign(v) * torch.floor(torch.abs(v) + 0.5) + zf
    mask = ((qr >= spec.q_min) & (qr <= spec.q_max)).to(torch.float64)
    if g == "per_token":
        return fq, mask
    if g == "per_channel":
        return fq.t().contiguous(), mask.t().contiguous()
    return fq.reshape(rows, cols), mask.reshape(rows, cols)


def _outlier_path(x_p, w_p, p_t, act_spec, weight_spec, cache, prefix, dv):  # layer.py:106-115
    torch = _torch()
    d = dv(p_t.scale)
    z = x_p * d[None, :]
    a, mask_a = _quantized(z, act_spec)
    b_pre = dv(w_p) / d[:, None]
    b, mask_b = _quantized(b_pre, weight_spec)
    cache[prefix] = {"x": x_p, "z": z, "a": a, "mask_a": mask_a, "b_pre": b_pre, "b": b, "mask_b": mask_b}
    if x_p.shape[1]:
        return a @ b
    return torch.zeros((x_p.shape[0], w_p.shape[1]), dtype=torch.float64, device=x_p.device)


def forward_with_cache(layer, batch, dev_cache=None):
    """layer.py:118-172 on the device: (y [T x d_out] fp64 CUDA, cache)."""
    torch = _torch()
    for name in ("p_main", "p_text", "p_vision"):
        if not getattr(getattr(layer, name), "is_diagonal", True):
            raise ValueError("dense transforms are not supported on the GPU path")
    dv = dev_cache or _Dev()
    p = layer.partition
    X = dv(batch.data)
    if X.shape[1] != p.dim:
        raise ValueError("batch width does not match partition dim")
    if not bool(torch.isfinite(X).all()):
        raise ValueError("non-finite value in matrix")
    tags = batch.tags.cpu().numpy() if _is_torch(batch.tags) else np.asarray(batch.tags)
    t_rows_np = np.flatnonzero(tags == 0)
    t_rows = torch.from_numpy(t_rows_np).to(X.device)
    idx = {k: torch.from_numpy(np.asarray(getattr(p, k), np.int64)).to(X.device)
           for k in ("c_main", "c_text", "c_vision")}
    x_m, x_t, x_v = X[:, idx["c_main"]], X[:, idx["c_text"]], X[:, idx["c_vision"]]
    act_aux = layer.act_spec.with_floor(layer.aux_bits_floor)
    w_aux = layer.weight_spec.with_floor(layer.aux_bits_floor)
    cache = {"text_rows": t_rows_np}

    y_t = _outlier_path(x_t, layer.w_text, layer.p_text, act_aux, w_aux, cache, "t", dv)
    y_v = _outlier_path(x_v, layer.w_vision, layer.p_vision, act_aux, w_aux, cache, "v", dv)

    d_m = dv(layer.p_main.scale)
    z = x_m * d_m[None, :]
    x_hat, mask_x = _quantized(z, layer.act_spec)
    w_prime = dv(layer.w_main) / d_m[:, None]
    cache["m"] = {"x": x_m, "z": z, "x_hat": x_hat, "mask_x": mask_x, "w_prime": w_prime}

    if layer.use_cws:
        br = layer.branch_smooth
        u = dv(br.u_star)
        v_eff = dv(br.gate)[:, None] * dv(br.v_base)
        r_pre = w_prime - u @ v_eff
        b_m, mask_r = _quantized(r_pre, layer.weight_spec)
        u_q, mask_u = _quantized(u, w_aux)
        v_q, mask_v = _quantized(v_eff, w_aux)
        y_m = x_hat @ b_m + (x_hat @ u_q) @ v_q
        cache["cws"] = {"r_pre": r_pre, "b_m": b_m, "mask_r": mask_r, "u_q": u_q, "mask_u": mask_u,
                        "v_q": v_q, "mask_v": mask_v, "v_eff": v_eff}
    else:
        b_m, mask_r = _quantized(w_prime, layer.weight_spec)
        y_m = x_hat @ b_m
        cache["main_w"] = {"b_m": b_m, "mask_r": mask_r}

    if layer.use_mac and t_rows_np.size:
        br = layer.branch_comp
        e_pre = (z - x_hat)[t_rows]
        e_q, mask_e = _quantized(e_pre, act_aux)
        uc_q, mask_uc = _quantized(dv(br.u_star), w_aux)
        vc_eff = dv(br.gate)[:, None] * dv(br.v_base)
        vc_q, mask_vc = _quantized(vc_eff, w_aux)
        comp = (e_q @ uc_q) @ vc_q
        y_m = y_m.clone()
        y_m[t_rows] += comp
        cache["mac"] = {"e_pre": e_pre, "e_q": e_q, "mask_e": mask_e, "uc_q": uc_q, "mask_uc": mask_uc,
                        "vc_q": vc_q, "mask_vc": mask_vc, "vc_eff": vc_eff}

    y = y_m + y_t + y_v
    return y, cache


# ------------------------------------------------------------------ calibration

def _param_layout(layer, cfg: CalibConfig):  # calibrate.py:69-94 (diagonal transforms)
    segments = []
    for name, learn, t in (("p_main", cfg.learn_p_main, layer.p_main),
                           ("p_text", cfg.learn_p_text, layer.p_text),
                           ("p_vision", cfg.learn_p_vision, layer.p_vision)):
        if learn and t.dim > 0:
            if not t.is_diagonal:
                raise ValueError("dense transforms are not supported on the GPU path")
            segments.append((name, t.dim))
    if cfg.learn_gates and layer.use_cws:
        segments.append(("gate_s", layer.branch_smooth.rank))
    if cfg.learn_gates and layer.use_mac:
        segments.append(("gate_c", layer.branch_comp.rank))
    return segments


def _initial_params(layer, segments) -> np.ndarray:  # calibrate.py:97-107
    parts = []
    for name, _size in segments:
        if name in ("p_main", "p_text", "p_vision"):
            parts.append(getattr(layer, name).log_scale)
        elif name == "gate_s":
            parts.append(layer.branch_smooth.gate)
        else:
            parts.append(layer.branch_comp.gate)
    return np.concatenate(parts) if parts else np.zeros(0)


def _apply_params(layer, segments, theta):  # calibrate.py:110-128
    from .layer import with_updated_params

    updates = {}
    offset = 0
    for name, size in segments:
        chunk = theta[offset: offset + size]
        offset += size
        if name in ("p_main", "p_text", "p_vision"):
            updates[name] = tr.diagonal_transform(np.exp(np.clip(chunk, _LOG_LO, _LOG_HI)))
        elif name == "gate_s":
            updates["gate_smooth"] = chunk.copy()
        else:
            updates["gate_comp"] = chunk.copy()
    return with_updated_params(layer, **updates)


def _loss(layer, batch, y_ref, dv):  # calibrate.py:128-131
    y, cache = forward_with_cache(layer, batch, dv)
    loss = float(((y - y_ref) ** 2).mean().item())
    return loss, y, cache


def _outlier_path_grad(path, d, g):  # calibrate.py:134-143
    dl_da = g @ path["b"].T
    dl_dz = path["mask_a"] * dl_da
    grad = (dl_dz * path["x"]).sum(0) * d
    dl_db = path["a"].T @ g
    dl_db_pre = path["mask_b"] * dl_db
    return grad - (dl_db_pre * path["b_pre"]).sum(1)


def analytic_gradient(layer, batch, segments, y_ref, dev_cache=None):
    """calibrate.py:146-222 on the device: (loss, flat gradient ndarray)."""
    torch = _torch()
    dv = dev_cache or _Dev()
    y_ref = dv(y_ref)
    loss, y, cache = _loss(layer, batch, y_ref, dv)
    g = (2.0 / y.numel()) * (y - y_ref)
    grads = {}
    names = {n for n, _ in segments}
    if "p_text" in names:
        grads["p_text"] = _outlier_path_grad(cache["t"], dv(layer.p_text.scale), g)
    if "p_vision" in names:
        grads["p_vision"] = _outlier_path_grad(cache["v"], dv(layer.p_vision.scale), g)
    m = cache["m"]
    t_rows = torch.from_numpy(cache["text_rows"]).to(g.device)
    need_main, need_gs, need_gc = "p_main" in names, "gate_s" in names, "gate_c" in names
    if need_main or need_gs or need_gc:
        if layer.use_cws:
            cws = cache["cws"]
            b_m, mask_r = cws["b_m"], cws["mask_r"]
            dl_dxhat = g @ b_m.T + (g @ cws["v_q"].T) @ cws["u_q"].T
        else:
            mw = cache["main_w"]
            b_m, mask_r = mw["b_m"], mw["mask_r"]
            dl_dxhat = g @ b_m.T
        dl_de_pre = None
        if layer.use_mac and "mac" in cache:
            mac = cache["mac"]
            dl_de_q = (g[t_rows] @ mac["vc_q"].T) @ mac["uc_q"].T
            dl_de_pre = mac["mask_e"] * dl_de_q
            dl_dxhat = dl_dxhat.clone()
            dl_dxhat[t_rows] -= dl_de_pre
        dl_dz = m["mask_x"] * dl_dxhat
        if dl_de_pre is not None:
            dl_dz = dl_dz.clone()
            dl_dz[t_rows] += dl_de_pre
        dl_db_m = m["x_hat"].T @ g
        dl_dr_pre = mask_r * dl_db_m
        if need_main:
            d = dv(layer.p_main.scale)
            grads["p_main"] = (dl_dz * m["x"]).sum(0) * d - (dl_dr_pre * m["w_prime"]).sum(1)
        if need_gs:
            cws = cache["cws"]
            br = layer.branch_smooth
            v_base = dv(br.v_base)
            dl_dv_q = (m["x_hat"] @ cws["u_q"]).T @ g
            dl_dv_eff = cws["mask_v"] * dl_dv_q
            grad_gs = (dl_dv_eff * v_base).sum(1)
            # the branch product is also subtracted inside the main residual
            grad_gs = grad_gs - torch.einsum("jk,jo,ko->k", dv(br.u_star), dl_dr_pre, v_base)
            grads["gate_s"] = grad_gs
        if need_gc:
            br = layer.branch_comp
            if "mac" in cache:
                mac = cache["mac"]
                dl_dvc_q = (mac["e_q"] @ mac["uc_q"]).T @ g[t_rows]
                dl_dvc_eff = mac["mask_vc"] * dl_dvc_q
                grads["gate_c"] = (dl_dvc_eff * dv(br.v_base)).sum(1)
            else:
                grads["gate_c"] = torch.zeros(br.rank, dtype=torch.float64, device=g.device)
    if not segments:
        return loss, np.zeros(0)
    return loss, torch.cat([grads[n] for n, _ in segments]).cpu().numpy()


def fd_gradient(layer, batch, segments, y_ref, theta, h, dev_cache=None):  # calibrate.py:225-240
    if theta.size > MAX_FD_PARAMS:
        raise ValueError(f"finite differences limited to {MAX_FD_PARAMS} parameters")
    dv = dev_cache or _Dev()
    y_ref = dv(y_ref)
    loss, _, _ = _loss(_apply_params(layer, segments, theta), batch, y_ref, dv)
    grad = np.zeros_like(theta)
    for i in range(theta.size):
        for sign in (1.0, -1.0):
            probe = theta.copy()
            probe[i] += sign * h
            l_probe, _, _ = _loss(_apply_params(layer, segments, probe), batch, y_ref, dv)
            grad[i] += sign * l_probe
        grad[i] /= 2.0 * h
    return loss, grad


def calibrate(layer, batch, cfg: CalibConfig):
    """calibrate.py:243-270 with the forward / gradient on the device."""
    dv = _Dev()
    segments = _param_layout(layer, cfg)
    y_ref = dv(batch.data) @ dv(layer.full_weight())  # forward_reference (layer.py:180-182)
    theta = _initial_params(layer, segments)
    trace = LossTrace()
    best_theta = theta.copy()
    best_loss = np.inf
    for step in range(cfg.steps):
        current = _apply_params(layer, segments, theta)
        if cfg.grad_mode == "analytic":
            loss, grad = analytic_gradient(current, batch, segments, y_ref, dv)
        else:
            loss, grad = fd_gradient(layer, batch, segments, y_ref, theta, cfg.fd_step, dv)
        if not np.isfinite(loss):
            raise NonFiniteLossError(step)
        trace.losses.append(loss)
        if loss < best_loss:
            best_loss = loss
            best_theta = theta.copy()
        if theta.size == 0:
            continue
        lr = cfg.learning_rate * 0.5 * (1.0 + np.cos(np.pi * step / cfg.steps))
        theta = theta - lr * grad
    return _apply_params(layer, segments, best_theta), trace
