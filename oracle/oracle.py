"""ctypes front-end of the CPU oracle (``oracle/liboracle.so``).

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (cpu_baseline leg and ``--impl reference``), always as the
checker or the timed CPU baseline -- never by the product package.

The C sources restate the reference functions named in ``vrp_oracle.h``;
this module only marshals numpy arrays.  The restatement is pinned to the
reference by ``tests/test_oracle_golden.py`` against ``tests/golden/``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"

OK, CAPACITY, DEADLOCK, MALFORMED = 0, 1, 2, 3


class PhiloxState(C.Structure):
    _fields_ = [("ctr", C.c_uint64 * 4), ("key", C.c_uint64 * 2), ("buffer", C.c_uint64 * 4),
                ("buffer_pos", C.c_int32), ("has_uint32", C.c_int32),
                ("uinteger", C.c_uint32), ("_pad", C.c_uint32)]

    @classmethod
    def from_numpy(cls, gen) -> "PhiloxState":
        st = gen.bit_generator.state
        if st["bit_generator"] != "Philox":
            raise TypeError("oracle RNG emulation needs Generator(Philox)")
        s = cls()
        for i in range(4):
            s.ctr[i] = int(st["state"]["counter"][i])
            s.buffer[i] = int(st["buffer"][i])
        for i in range(2):
            s.key[i] = int(st["state"]["key"][i])
        s.buffer_pos = int(st["buffer_pos"])
        s.has_uint32 = int(st["has_uint32"])
        s.uinteger = int(st["uinteger"])
        return s

    def to_numpy_state(self) -> dict:
        return {
            "bit_generator": "Philox",
            "state": {"counter": np.array(list(self.ctr), dtype=np.uint64),
                      "key": np.array(list(self.key), dtype=np.uint64)},
            "buffer": np.array(list(self.buffer), dtype=np.uint64),
            "buffer_pos": int(self.buffer_pos),
            "has_uint32": int(self.has_uint32),
            "uinteger": int(self.uinteger),
        }


_lib = None


def build() -> Path:
    """Compile liboracle.so in place (plain C, gcc)."""
    env = dict(os.environ)
    cc = "/usr/bin/gcc" if Path("/usr/bin/gcc").exists() else env.get("CC", "gcc")
    subprocess.run(["make", "-s", "-C", str(HERE), f"CC={cc}"], check=True, env=env)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        P = C.c_void_p
        i32, i64, f64 = C.c_int32, C.c_int64, C.c_double
        L.orc_makespan_batch.argtypes = [i32, i32, i32, P, P, P, P, i64, i32, P, P, P, i32]
        L.orc_makespan_batch.restype = None
        L.orc_evaluate.argtypes = [i32, i32, i32, P, P, P, P, P, P, P, P, P]
        L.orc_evaluate.restype = C.c_int
        L.orc_decode_batch.argtypes = [i32, i32, i32, P, P, P, i64, i32, f64, P, P, P, P, P, P, i32]
        L.orc_decode_batch.restype = None
        L.orc_evolve.argtypes = [P, P, i64, i64, f64, f64, f64, C.POINTER(PhiloxState), P]
        L.orc_evolve.restype = C.c_int
        L.orc_stable_argsort.argtypes = [P, i64, P]
        L.orc_hint_vehicle.argtypes = [i32, f64]
        L.orc_hint_vehicle.restype = i32
        L.orc_philox_next64.argtypes = [C.POINTER(PhiloxState)]
        L.orc_philox_next64.restype = C.c_uint64
        L.orc_philox_next_double.argtypes = [C.POINTER(PhiloxState)]
        L.orc_philox_next_double.restype = f64
        L.orc_philox_integers.argtypes = [C.POINTER(PhiloxState), C.c_uint64]
        L.orc_philox_integers.restype = C.c_uint64
        L.orc_default_threads.restype = i32
        L.orc_py_sum.argtypes = [P, C.c_int]
        L.orc_py_sum.restype = f64
        L.orc_reinsert_all.argtypes = [i32, i32, i32, P, P, P, P, P, i32, i32, C.POINTER(PhiloxState)]
        L.orc_reinsert_all.restype = C.c_int
        L.orc_remove_customers.argtypes = [i32, i32, i32, P, P, P, i32, P]
        L.orc_remove_customers.restype = C.c_int
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _inst(inst):
    """(n, m, k, d, p) from anything with those attributes or a tuple."""
    if isinstance(inst, tuple):
        n, m, k, d, p = inst
    else:
        n, m, k = inst.n, inst.m, inst.k
        d, p = inst.d, inst.p
    d = np.ascontiguousarray(np.asarray(d, dtype=np.float64)).reshape(n + 1, n + 1)
    p = np.ascontiguousarray(np.asarray(p, dtype=np.float64)).reshape(n + 1)
    return int(n), int(m), int(k), d, p


def makespan_batch(inst, ops, lens, mode="exact", threads=0, want_returns=False):
    """mode: 'exact' (schedule.exact_makespan), 'evaluate' (schedule.evaluate),
    'two_pass' (schedule.two_pass_estimate).  ops: int32 [N, 2n] vehicle-major,
    lens: int32 [N, m].  Returns (z, status[, returns])."""
    n, m, k, d, p = _inst(inst)
    ops = np.ascontiguousarray(ops, dtype=np.int32).reshape(-1, 2 * n)
    lens = np.ascontiguousarray(lens, dtype=np.int32).reshape(-1, m)
    N = ops.shape[0]
    z = np.zeros(N, np.float64)
    st = np.zeros(N, np.int32)
    ret = np.zeros((N, m), np.float64) if want_returns else None
    code = {"exact": 0, "evaluate": 1, "two_pass": 2}[mode]
    lib().orc_makespan_batch(n, m, k, _ptr(d), _ptr(p), _ptr(ops), _ptr(lens), N, code,
                             _ptr(z), _ptr(st), _ptr(ret), int(threads))
    return (z, st, ret) if want_returns else (z, st)


def evaluate_one(inst, ops, lens):
    """Full-record evaluate: (status, z, returns[m], arrival[2n], time[2n], q0[m])."""
    n, m, k, d, p = _inst(inst)
    ops = np.ascontiguousarray(ops, dtype=np.int32).reshape(2 * n)
    lens = np.ascontiguousarray(lens, dtype=np.int32).reshape(m)
    z = np.zeros(1)
    ret = np.zeros(m)
    arr = np.zeros(2 * n)
    tim = np.zeros(2 * n)
    q0 = np.zeros(m, np.int32)
    st = lib().orc_evaluate(n, m, k, _ptr(d), _ptr(p), _ptr(ops), _ptr(lens), _ptr(z),
                            _ptr(ret), _ptr(arr), _ptr(tim), _ptr(q0))
    return st, float(z[0]), ret, arr, tim, q0


def decode_batch(inst, genes, relax=True, penalty=1e6, threads=0):
    """brkga.decode over rows of genes [N, 4n] -> dict of arrays."""
    n, m, k, d, p = _inst(inst)
    genes = np.ascontiguousarray(genes, dtype=np.float64).reshape(-1, 4 * n)
    N = genes.shape[0]
    out = {
        "ops": np.zeros((N, 2 * n), np.int32),
        "lens": np.zeros((N, m), np.int32),
        "fitness": np.zeros(N),
        "makespan": np.zeros(N),
        "scheduled": np.zeros(N, np.int32),
        "visits": np.zeros(N, np.int64),
    }
    lib().orc_decode_batch(n, m, k, _ptr(d), _ptr(p), _ptr(genes), N, int(bool(relax)),
                           float(penalty), _ptr(out["ops"]), _ptr(out["lens"]),
                           _ptr(out["fitness"]), _ptr(out["makespan"]), _ptr(out["scheduled"]),
                           _ptr(out["visits"]), int(threads))
    return out


def evolve(population, fitness, elite_fraction, mutant_fraction, elite_bias, gen):
    """brkga.evolve with a numpy Generator(Philox); advances ``gen`` exactly as
    the reference would.  Raises ValueError for PopulationTooSmall."""
    pop = np.ascontiguousarray(population, dtype=np.float64)
    fit = np.ascontiguousarray(fitness, dtype=np.float64)
    N, G = pop.shape
    st = PhiloxState.from_numpy(gen)
    out = np.empty_like(pop)
    rc = lib().orc_evolve(_ptr(pop), _ptr(fit), N, G, float(elite_fraction),
                          float(mutant_fraction), float(elite_bias), C.byref(st), _ptr(out))
    if rc != 0:
        raise ValueError("population too small")
    gen.bit_generator.state = st.to_numpy_state()
    return out


def stable_argsort(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    order = np.empty(x.shape[0], np.int64)
    lib().orc_stable_argsort(_ptr(x), x.shape[0], _ptr(order))
    return order


def default_threads() -> int:
    return int(lib().orc_default_threads())


def remove_customers(inst, ops, lens, customers):
    """insertion.remove_customers: (ops, lens, removed sorted)."""
    n, m, k, d, p = _inst(inst)
    ops = np.array(ops, dtype=np.int32).reshape(-1).copy()
    full = np.full(max(2 * n, ops.size), -1, np.int32)
    full[:ops.size] = ops
    lens = np.array(lens, dtype=np.int32).copy()
    cust = np.ascontiguousarray(customers, dtype=np.int32)
    out = np.zeros(n, np.int32)
    cnt = lib().orc_remove_customers(n, m, k, _ptr(full), _ptr(lens), _ptr(cust), cust.size, _ptr(out))
    return full, lens, out[:cnt].copy()


def reinsert_all(inst, ops, lens, removed, regret_k=0, gen=None):
    """insertion.reinsert_all on a fresh InsertionContext(partial): returns
    (status, ops, lens); status 1 = RepairFailed.  ``gen`` (Generator(Philox)
    or None) is advanced like the reference's rng."""
    n, m, k, d, p = _inst(inst)
    full = np.full(2 * n, -1, np.int32)
    ops = np.asarray(ops, dtype=np.int32).reshape(-1)
    lens = np.array(lens, dtype=np.int32).copy()
    full[:int(lens.sum())] = ops[:int(lens.sum())]
    rem = np.ascontiguousarray(removed, dtype=np.int32)
    st = None
    if gen is not None:
        st = PhiloxState.from_numpy(gen)
    rc = lib().orc_reinsert_all(n, m, k, _ptr(d), _ptr(p), _ptr(full), _ptr(lens), _ptr(rem),
                                rem.size, int(regret_k), C.byref(st) if st is not None else None)
    if gen is not None:
        gen.bit_generator.state = st.to_numpy_state()
    return rc, full, lens


def py_sum(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    return float(lib().orc_py_sum(_ptr(x), x.size))
