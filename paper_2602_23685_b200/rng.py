"""Bridge between numpy's ``Generator(Philox)`` and the device RNG state.

The device kernels (``vrp_evolve``; later the ALNS operators) consume the
numpy Philox stream bit for bit (see csrc/evolve.cu): the state struct
``vrp_philox`` in include/vrp_rpd.h is field-for-field
``Generator(Philox).bit_generator.state``.  These helpers move that state to
a device buffer and back, so a caller's generator continues exactly where
numpy's would.

The reference's own drivers seed ``Generator(PCG64(seed))``
(brkga.py:436, alns.py:495-496).  PCG64 is not counter-based, so the device
paths use ``Generator(Philox(key=(seed, stream_tag)))`` instead: the same
algorithm over a different (equally uniform) stream.  Parity tests inject
the same Philox generator into the reference (tests/golden/make_golden.py).
"""
from __future__ import annotations

import numpy as np
import torch

_DTYPE = np.dtype([("ctr", "<u8", 4), ("key", "<u8", 2), ("buffer", "<u8", 4),
                   ("buffer_pos", "<i4"), ("has_uint32", "<i4"), ("uinteger", "<u4"),
                   ("reserved", "<u4")])
assert _DTYPE.itemsize == 96

BRKGA_STREAM = 0xB4C6A  # Philox key[1] used by run_brkga(seed)
ALNS_STREAM = 0xA1B5


def philox_generator(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=(int(seed) & (2**64 - 1), int(stream))))


def as_philox(rng, stream: int = 0) -> np.random.Generator:
    """The generator itself when it is a Generator(Philox); otherwise a Philox
    generator keyed by two words drawn from ``rng`` (documented divergence)."""
    if isinstance(rng, np.random.Generator) and isinstance(rng.bit_generator, np.random.Philox):
        return rng
    if rng is None:
        return philox_generator(0, stream)
    if isinstance(rng, (int, np.integer)):
        return philox_generator(int(rng), stream)
    words = rng.integers(0, 2**63, size=2)
    return np.random.Generator(np.random.Philox(key=(int(words[0]), int(words[1]) ^ stream)))


def state_bytes(gen: np.random.Generator) -> np.ndarray:
    """The vrp_philox struct (uint8[96]) of a Generator(Philox)."""
    st = gen.bit_generator.state
    if st["bit_generator"] != "Philox":
        raise TypeError("device RNG needs Generator(Philox)")
    rec = np.zeros(1, dtype=_DTYPE)
    rec["ctr"][0] = np.asarray(st["state"]["counter"], dtype=np.uint64)
    rec["key"][0] = np.asarray(st["state"]["key"], dtype=np.uint64)
    rec["buffer"][0] = np.asarray(st["buffer"], dtype=np.uint64)
    rec["buffer_pos"][0] = int(st["buffer_pos"])
    rec["has_uint32"][0] = int(st["has_uint32"])
    rec["uinteger"][0] = int(st["uinteger"])
    return rec.view(np.uint8).copy()


def set_state_bytes(gen: np.random.Generator, raw) -> None:
    """Load a vrp_philox struct (uint8[96]) into a Generator(Philox)."""
    rec = np.ascontiguousarray(raw, dtype=np.uint8).reshape(-1).view(_DTYPE)[0]
    gen.bit_generator.state = {
        "bit_generator": "Philox",
        "state": {"counter": np.array(rec["ctr"], dtype=np.uint64),
                  "key": np.array(rec["key"], dtype=np.uint64)},
        "buffer": np.array(rec["buffer"], dtype=np.uint64),
        "buffer_pos": int(rec["buffer_pos"]),
        "has_uint32": int(rec["has_uint32"]),
        "uinteger": int(rec["uinteger"]),
    }


def state_to_device(gen: np.random.Generator, device=None) -> torch.Tensor:
    t = torch.from_numpy(state_bytes(gen))
    return t.to(device if device is not None else torch.device("cuda", torch.cuda.current_device()))


def state_from_device(gen: np.random.Generator, t: torch.Tensor) -> None:
    set_state_bytes(gen, t.detach().cpu().numpy())


def random_device(gen: np.random.Generator, shape, device=None) -> torch.Tensor:
    """``gen.random(shape)`` generated on the device (vrp_random_fill): the
    same doubles in the same order, and ``gen`` advanced exactly as numpy
    would advance it."""
    from . import _native as N
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    count = int(np.prod(shape))
    out = torch.empty(tuple(shape), dtype=torch.float64, device=dev)
    st = state_to_device(gen, dev)
    N.check(N.lib().vrp_random_fill(N.ptr(st), count, N.ptr(out), N.stream_handle()), "vrp_random_fill")
    state_from_device(gen, st)
    return out
