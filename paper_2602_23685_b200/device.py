"""Device-resident instances and the batched entry points (torch tensors in,
torch tensors out), all routed through the C-ABI of include/vrp_rpd.h.

Batch layout (shared with the C-ABI and the oracle):
  ops   int16|int32 [N, 2n]  op code 2(c-1)+kind, routes concatenated vehicle-major
  lens  int32 [N, m]         route lengths
  genes fp64  [N, 4n]        BRKGA chromosomes (priorities | hints)
"""
from __future__ import annotations

import ctypes as C
import weakref

import numpy as np
import torch

from . import _native as N

_HANDLES: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


class DeviceInstance:
    """Owns the device copy of an instance (d fp64 + int32 twin, p) on the
    current CUDA device.  Create via :func:`device_instance`."""

    def __init__(self, n: int, m: int, k: int, d: np.ndarray, p: np.ndarray):
        L = N.lib()
        d = np.ascontiguousarray(d, dtype=np.float64)
        p = np.ascontiguousarray(p, dtype=np.float64)
        if d.shape != (n + 1, n + 1) or p.shape != (n + 1,):
            raise ValueError("d must be (n+1)x(n+1) and p (n+1)")
        h = C.c_void_p()
        N.check(L.vrp_instance_create(n, m, k, d.ctypes.data_as(C.c_void_p),
                                      p.ctypes.data_as(C.c_void_p), C.byref(h)),
                "vrp_instance_create")
        self._h = h
        self.n, self.m, self.k = n, m, k
        self.device = torch.cuda.current_device()
        integral = C.c_int32()
        N.check(L.vrp_instance_info(h, None, None, None, C.byref(integral)))
        self.integral = bool(integral.value)

    @property
    def handle(self):
        return self._h

    def __del__(self):
        try:
            h = getattr(self, "_h", None)
            if h is not None and N._lib is not None:
                N._lib.vrp_instance_destroy(h)
            self._h = None
        except Exception:  # interpreter shutdown: module globals already gone
            pass


def device_instance(instance) -> DeviceInstance:
    """Cached DeviceInstance for an ``Instance`` (or anything with n,m,k,d,p)."""
    N.lib()  # raises NativeUnavailable without the library or a device
    dev = torch.cuda.current_device()
    cache = getattr(instance, "_cache", None)
    key = ("device_instance", dev)
    if cache is not None and key in cache:
        return cache[key]
    if hasattr(instance, "arrays"):
        d, p = instance.arrays()
    else:
        d, p = np.asarray(instance.d, np.float64), np.asarray(instance.p, np.float64)
    di = DeviceInstance(int(instance.n), int(instance.m), int(instance.k), d, p)
    if cache is not None:
        cache[key] = di
    return di


def _check_out(res, dev, **spec):
    """Caller-supplied output tensors must match the batch (the kernels write
    through their raw pointers)."""
    for name, (shape, dtype) in spec.items():
        t = res.get(name)
        if t is None:
            continue
        if tuple(t.shape) != tuple(shape) or t.dtype != dtype or t.device != dev or not t.is_contiguous():
            raise ValueError(f"out[{name!r}] must be a contiguous {dtype} tensor of shape {tuple(shape)} on {dev}, "
                             f"got {t.dtype} {tuple(t.shape)} on {t.device}")


def row_stride(t) -> int:
    """Elements between rows; a size-1 leading dim may report any stride."""
    return int(t.stride(0)) if t.shape[0] > 1 else int(t.shape[1])


def _cuda(t, dtype=None):
    t = torch.as_tensor(t)
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    if not t.is_cuda:
        t = t.cuda()
    return t.contiguous()


def makespan_batch(instance, ops, lens, mode: int = N.MODE_EXACT, want_returns: bool = False,
                   want_bottleneck: bool = False, stream=None, out=None):
    """Score a batch of candidates on the GPU (K1/K2).

    ``mode``: 0 exact_makespan, 1 evaluate (validating), 2 two_pass_estimate.
    Returns dict of device tensors: z fp64 [N], status int32 [N] (+ returns
    fp64 [N, m], bottleneck int32 [N])."""
    di = device_instance(instance)
    ops = _cuda(ops)
    if ops.dtype not in (torch.int16, torch.int32):
        ops = ops.to(torch.int32)
    lens = _cuda(lens, torch.int32)
    if ops.dim() == 1:
        ops = ops.unsqueeze(0)
    if lens.dim() == 1:
        lens = lens.unsqueeze(0)
    Nc = ops.shape[0]
    if lens.shape != (Nc, di.m):
        raise ValueError(f"lens must be [N, m={di.m}], got {tuple(lens.shape)}")
    dev = ops.device
    res = out if out is not None else {}
    if "z" not in res:
        res["z"] = torch.empty(Nc, dtype=torch.float64, device=dev)
        res["status"] = torch.empty(Nc, dtype=torch.int32, device=dev)
    if want_returns and "returns" not in res:
        res["returns"] = torch.empty((Nc, di.m), dtype=torch.float64, device=dev)
    if want_bottleneck and "bottleneck" not in res:
        res["bottleneck"] = torch.empty(Nc, dtype=torch.int32, device=dev)
    _check_out(res, dev, z=((Nc,), torch.float64), status=((Nc,), torch.int32),
               returns=((Nc, di.m), torch.float64), bottleneck=((Nc,), torch.int32))
    L = N.lib()
    N.check(L.vrp_makespan_batch(di.handle, N.ptr(ops), ops.element_size(), row_stride(ops),
                                 N.ptr(lens), Nc, int(mode), N.ptr(res["z"]), N.ptr(res["status"]),
                                 N.ptr(res.get("returns")), N.ptr(res.get("bottleneck")),
                                 N.stream_handle(stream)), "vrp_makespan_batch")
    return res


def evaluate_records(instance, ops, lens, stream=None):
    """Full evaluate records (arrival/time per op, q0 per vehicle) for a batch."""
    di = device_instance(instance)
    ops = _cuda(ops, torch.int32)
    lens = _cuda(lens, torch.int32)
    if ops.dim() == 1:
        ops, lens = ops.unsqueeze(0), lens.unsqueeze(0)
    Nc = ops.shape[0]
    dev = ops.device
    res = {"z": torch.empty(Nc, dtype=torch.float64, device=dev),
           "status": torch.empty(Nc, dtype=torch.int32, device=dev),
           "returns": torch.empty((Nc, di.m), dtype=torch.float64, device=dev),
           # defined for status-OK candidates (every op executed), like the
           # reference's Schedule, which only exists for those
           "arrival": torch.empty(ops.shape, dtype=torch.float64, device=dev),
           "time": torch.empty(ops.shape, dtype=torch.float64, device=dev),
           "q0": torch.empty((Nc, di.m), dtype=torch.int32, device=dev)}
    N.check(N.lib().vrp_evaluate_records(di.handle, N.ptr(ops), row_stride(ops), N.ptr(lens), Nc,
                                         N.ptr(res["z"]), N.ptr(res["status"]),
                                         N.ptr(res["returns"]), N.ptr(res["arrival"]),
                                         N.ptr(res["time"]), N.ptr(res["q0"]),
                                         N.stream_handle(stream)), "vrp_evaluate_records")
    return res


def decode_batch(instance, genes, relax: bool = True, penalty: float = 1e6,
                 want_solution: bool = True, op_dtype=torch.int32, stream=None, out=None):
    """BRKGA decode (K3) of genes [N, 4n] fp64 on the GPU.

    Returns dict of device tensors: fitness, makespan, scheduled, visits and,
    if ``want_solution``, ops [N, 2n] (vehicle-major, -1 padded) and lens [N, m]."""
    di = device_instance(instance)
    genes = _cuda(genes, torch.float64)
    if genes.dim() == 1:
        genes = genes.unsqueeze(0)
    Nc = genes.shape[0]
    if genes.shape[1] < 4 * di.n:
        raise ValueError(f"chromosomes need 4n = {4 * di.n} genes")
    dev = genes.device
    res = out if out is not None else {}
    if "fitness" not in res:
        res["fitness"] = torch.empty(Nc, dtype=torch.float64, device=dev)
        res["makespan"] = torch.empty(Nc, dtype=torch.float64, device=dev)
        res["scheduled"] = torch.empty(Nc, dtype=torch.int32, device=dev)
        res["visits"] = torch.empty(Nc, dtype=torch.int64, device=dev)
    if want_solution and "ops" not in res:
        res["ops"] = torch.empty((Nc, 2 * di.n), dtype=op_dtype, device=dev)
        res["lens"] = torch.empty((Nc, di.m), dtype=torch.int32, device=dev)
    _check_out(res, dev, fitness=((Nc,), torch.float64), makespan=((Nc,), torch.float64),
               scheduled=((Nc,), torch.int32), visits=((Nc,), torch.int64), lens=((Nc, di.m), torch.int32))
    if want_solution:
        o = res["ops"]
        if o.dim() != 2 or o.shape[0] != Nc or o.shape[1] < 2 * di.n or o.dtype not in (torch.int16, torch.int32) \
                or o.device != dev:
            raise ValueError(f"out['ops'] must be int16/int32 [N={Nc}, >=2n] on {dev}")
    ops = res.get("ops") if want_solution else None
    N.check(N.lib().vrp_decode_batch(
        di.handle, N.ptr(genes), row_stride(genes), Nc, int(bool(relax)), float(penalty),
        N.ptr(res["fitness"]), N.ptr(res["makespan"]), N.ptr(res["scheduled"]),
        N.ptr(res["visits"]), N.ptr(ops), ops.element_size() if ops is not None else 4,
        row_stride(ops) if ops is not None else 2 * di.n,
        N.ptr(res.get("lens") if want_solution else None), N.stream_handle(stream)),
        "vrp_decode_batch")
    return res


N_STREAMS = 2  # copy/compute streams of score_host_batch


def _pipeline(di, chunk: int, op_dtype):
    # held by the DeviceInstance (one device each), so the buffers live exactly
    # as long as the instance
    pipes = di.__dict__.setdefault("_pipes", {})
    key = (chunk, op_dtype, N_STREAMS)
    st = pipes.get(key)
    if st is None:
        dev = torch.device("cuda", torch.cuda.current_device())
        st = {"streams": [torch.cuda.Stream(device=dev) for _ in range(N_STREAMS)],
              "bufs": [{"ops": torch.empty((chunk, 2 * di.n), dtype=op_dtype, device=dev),
                        "lens": torch.empty((chunk, di.m), dtype=torch.int32, device=dev),
                        "z": torch.empty(chunk, dtype=torch.float64, device=dev),
                        "status": torch.empty(chunk, dtype=torch.int32, device=dev)}
                       for _ in range(N_STREAMS)]}
        pipes[key] = st
    return st


def score_host_batch(instance, ops, lens, mode: int = N.MODE_EXACT, chunk: int = 1 << 14):
    """End-to-end scoring of HOST candidates: chunks are copied host->device,
    scored by K1/K2 and their (z, status) copied back, alternating two CUDA
    streams so the PCIe transfers overlap the kernel.  ``ops``/``lens`` should
    be pinned CPU tensors (numpy arrays are pinned on the fly).  Returns numpy
    (z, status)."""
    di = device_instance(instance)
    if not isinstance(ops, torch.Tensor):
        ops = torch.from_numpy(np.ascontiguousarray(ops)).pin_memory()
    if not isinstance(lens, torch.Tensor):
        lens = torch.from_numpy(np.ascontiguousarray(lens, dtype=np.int32)).pin_memory()
    if ops.dtype not in (torch.int16, torch.int32):
        ops = ops.to(torch.int32)
    Nc = ops.shape[0]
    z = torch.empty(Nc, dtype=torch.float64, pin_memory=True)
    status = torch.empty(Nc, dtype=torch.int32, pin_memory=True)
    st = _pipeline(di, chunk, ops.dtype)
    cur = torch.cuda.current_stream()
    for s in st["streams"]:
        s.wait_stream(cur)
    for i, a in enumerate(range(0, Nc, chunk)):
        b = min(Nc, a + chunk)
        c = b - a
        s, buf = st["streams"][i % len(st["streams"])], st["bufs"][i % len(st["bufs"])]
        with torch.cuda.stream(s):
            buf["ops"][:c].copy_(ops[a:b], non_blocking=True)
            buf["lens"][:c].copy_(lens[a:b], non_blocking=True)
            out = {"z": buf["z"][:c], "status": buf["status"][:c]}
            makespan_batch(instance, buf["ops"][:c], buf["lens"][:c], mode=mode, stream=s, out=out)
            z[a:b].copy_(buf["z"][:c], non_blocking=True)
            status[a:b].copy_(buf["status"][:c], non_blocking=True)
    for s in st["streams"]:
        cur.wait_stream(s)
    cur.synchronize()
    return z.numpy(), status.numpy()


def repair_batch(instance, partial_ops, partial_lens, removed, nremoved, regret_k, states=None,
                 stream=None):
    """K5: reinsert_all on N partial solutions (device tensors in/out).

    partial_ops [N, >=2n] int32, partial_lens [N, m] int32, removed [N, R] int32
    (customers), nremoved [N] int32, regret_k [N] int32, states: uint8 [N, 96]
    device generator states (advanced in place) or None (deterministic).
    Returns dict(ops [N, 2n], lens [N, m], status [N]) -- status 0 OK,
    1 RepairFailed, 2 malformed input."""
    di = device_instance(instance)
    po = _cuda(partial_ops, torch.int32)
    pl = _cuda(partial_lens, torch.int32)
    rm = _cuda(removed, torch.int32)
    nr = _cuda(nremoved, torch.int32)
    rk = _cuda(regret_k, torch.int32)
    Nn = po.shape[0]
    dev = po.device
    out = {"ops": torch.empty((Nn, 2 * di.n), dtype=torch.int32, device=dev),
           "lens": torch.empty((Nn, di.m), dtype=torch.int32, device=dev),
           "status": torch.empty(Nn, dtype=torch.int32, device=dev)}
    if states is not None and (states.dtype != torch.uint8 or states.shape[-1] != 96):
        raise ValueError("states must be uint8 [N, 96] device generator states")
    N.check(N.lib().vrp_repair_batch(di.handle, N.ptr(po), row_stride(po), N.ptr(pl), N.ptr(rm),
                                     row_stride(rm) if rm.dim() == 2 else 0, N.ptr(nr), N.ptr(rk),
                                     N.ptr(states), N.ptr(out["ops"]), 2 * di.n, N.ptr(out["lens"]),
                                     N.ptr(out["status"]), Nn, N.stream_handle(stream)),
            "vrp_repair_batch")
    return out


DESTROY_CODES = {"random": 0, "worst": 1, "shaw": 2, "cluster": 3, "route": 4, "critical_path": 5}


def destroy_batch(instance, ops, lens, operators, q, q_min, states, stream=None):
    """K6: destroy + remove_customers on N complete solutions (device tensors).

    ops [N, >=2n] int32, lens [N, m] int32, operators [N] int32 (DESTROY_CODES),
    q [N] int32, states uint8 [N, 96] device generators (advanced in place).
    Returns dict(ops [N, 2n] partials, lens [N, m], removed [N, n] (sorted,
    -padded after nremoved), nremoved [N])."""
    di = device_instance(instance)
    o = _cuda(ops, torch.int32)
    ln = _cuda(lens, torch.int32)
    op = _cuda(operators, torch.int32)
    qq = _cuda(q, torch.int32)
    Nn = o.shape[0]
    dev = o.device
    if states.dtype != torch.uint8 or states.shape[-1] != 96 or states.shape[0] != Nn:
        raise ValueError("states must be uint8 [N, 96] device generator states")
    out = {"ops": torch.empty((Nn, 2 * di.n), dtype=torch.int32, device=dev),
           "lens": torch.empty((Nn, di.m), dtype=torch.int32, device=dev),
           "removed": torch.zeros((Nn, di.n), dtype=torch.int32, device=dev),
           "nremoved": torch.empty(Nn, dtype=torch.int32, device=dev)}
    N.check(N.lib().vrp_destroy_batch(di.handle, N.ptr(o), row_stride(o), N.ptr(ln), N.ptr(op), N.ptr(qq),
                                      int(q_min), N.ptr(states), N.ptr(out["ops"]), 2 * di.n,
                                      N.ptr(out["lens"]), N.ptr(out["removed"]), di.n,
                                      N.ptr(out["nremoved"]), Nn, N.stream_handle(stream)),
            "vrp_destroy_batch")
    return out


def remove_batch(instance, ops, lens, picked, npicked, stream=None):
    """insertion.remove_customers on N solutions (vrp_remove_batch, K6's
    removal + capacity cascade).  ops [N, >=2n] / lens [N, m] int32, picked
    [N, P] int32 customers with npicked [N] valid per row.  Returns dict(ops
    [N, 2n] partials, lens [N, m], removed [N, n] sorted, nremoved [N])."""
    di = device_instance(instance)
    o = _cuda(ops, torch.int32)
    ln = _cuda(lens, torch.int32)
    pk = _cuda(picked, torch.int32)
    npk = _cuda(npicked, torch.int32)
    if o.dim() == 1:
        o, ln = o.unsqueeze(0), ln.unsqueeze(0)
    if pk.dim() == 1:
        pk = pk.unsqueeze(0)
    Nn = o.shape[0]
    if ln.shape != (Nn, di.m) or pk.shape[0] != Nn or npk.shape != (Nn,):
        raise ValueError("remove_batch: ops/lens/picked/npicked shapes disagree")
    dev = o.device
    out = {"ops": torch.empty((Nn, 2 * di.n), dtype=torch.int32, device=dev),
           "lens": torch.empty((Nn, di.m), dtype=torch.int32, device=dev),
           "removed": torch.zeros((Nn, di.n), dtype=torch.int32, device=dev),
           "nremoved": torch.empty(Nn, dtype=torch.int32, device=dev)}
    N.check(N.lib().vrp_remove_batch(di.handle, N.ptr(o), row_stride(o), N.ptr(ln), N.ptr(pk),
                                     row_stride(pk), N.ptr(npk), N.ptr(out["ops"]), 2 * di.n,
                                     N.ptr(out["lens"]), N.ptr(out["removed"]), di.n,
                                     N.ptr(out["nremoved"]), Nn, N.stream_handle(stream)),
            "vrp_remove_batch")
    return out


def removal_gains_batch(instance, ops, lens, stream=None):
    """insertion.removal_gains on N complete solutions (vrp_removal_gains):
    fp64 [N, n+1] device tensor, column c = gain of customer c (column 0 = 0)."""
    di = device_instance(instance)
    o = _cuda(ops, torch.int32)
    ln = _cuda(lens, torch.int32)
    if o.dim() == 1:
        o, ln = o.unsqueeze(0), ln.unsqueeze(0)
    Nn = o.shape[0]
    if ln.shape != (Nn, di.m):
        raise ValueError(f"lens must be [N, m={di.m}]")
    gains = torch.empty((Nn, di.n + 1), dtype=torch.float64, device=o.device)
    N.check(N.lib().vrp_removal_gains(di.handle, N.ptr(o), row_stride(o), N.ptr(ln), N.ptr(gains),
                                      di.n + 1, Nn, N.stream_handle(stream)), "vrp_removal_gains")
    return gains


# vrp_alns_worker / vrp_alns_params (include/vrp_rpd.h), field for field
ALNS_WORKER_DTYPE = np.dtype([
    ("rng", np.uint8, 96), ("z", "<f8"), ("z_best", "<f8"), ("temperature", "<f8"), ("t_init", "<f8"),
    ("weights", "<f8", 10), ("scores", "<f8", 10), ("attempts", "<i8", 10),
    ("stagnation", "<i8"), ("accepted", "<i8"), ("rejected", "<i8"), ("reheats", "<i8"),
    ("best_it", "<i8"), ("n_trace", "<i4"), ("n_rows", "<i4")])


class AlnsParamsC(C.Structure):
    _fields_ = [("t0", C.c_double), ("alpha", C.c_double), ("reheat_factor", C.c_double),
                ("reaction", C.c_double), ("sigma1", C.c_double), ("sigma2", C.c_double),
                ("sigma3", C.c_double), ("min_weight", C.c_double),
                ("stagnation_threshold", C.c_int64), ("weight_interval", C.c_int64),
                ("q_min", C.c_int32), ("reserved", C.c_int32)]


def alns_iterate(instance, params: AlnsParamsC, workers, cur_ops, cur_lens, best_ops, best_lens,
                 q_draws, it_begin: int, it_end: int, trace_it, trace_z, rows_it, rows_val,
                 stream=None):
    """Device-resident ALNS iterations it_begin..it_end for every worker
    (vrp_alns_iterate).  All tensors live on the device and are updated in place:
    workers uint8 [W, 416], cur/best ops [W, 2n] + lens [W, m], q_draws [W, >=it_end],
    trace_it/trace_z [W, cap], rows_it [W, rcap], rows_val [W, rcap, 12]."""
    di = device_instance(instance)
    W = workers.shape[0]
    N.check(N.lib().vrp_alns_iterate(
        di.handle, C.byref(params), N.ptr(workers), W, N.ptr(cur_ops), N.ptr(cur_lens),
        N.ptr(best_ops), N.ptr(best_lens), N.ptr(q_draws), row_stride(q_draws), int(it_begin), int(it_end),
        N.ptr(trace_it), N.ptr(trace_z), trace_it.shape[1], N.ptr(rows_it), N.ptr(rows_val),
        rows_it.shape[1], N.stream_handle(stream)), "vrp_alns_iterate")
