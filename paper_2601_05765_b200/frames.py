"""Frame persistence and warm start (cli_io write_frame /
read_frame).

Little-endian binary: magic "POTF", format version u32, n u64, step u64,
time f64, then the arrays as f64 in declared order -- positions [n,3],
velocities [n,3], weights psi [n], cell volumes [n], free-surface areas [n],
phase ids [n] -- then the footer worst_rel_error f64, newton_iters u64,
wall_ms f64, and a CRC32 (zlib) of everything before it.
"""
from __future__ import annotations

import struct
import zlib
from dataclasses import dataclass

import numpy as np

MAGIC = b"POTF"
VERSION = 1
_HEAD = struct.Struct("<4sIQQd")
_FOOT = struct.Struct("<dQd")


class FrameError(ValueError):
    """Bad magic / version / size."""


class CrcError(FrameError):
    """CRC32 mismatch (corrupted or truncated frame)."""


@dataclass
class FrameRecord:
    step: int
    time: float
    x: np.ndarray       # [n,3]
    v: np.ndarray       # [n,3]
    psi: np.ndarray     # [n]
    vol: np.ndarray     # [n]
    ksur: np.ndarray    # [n]
    phase: np.ndarray   # [n]
    worst_rel_error: float = 0.0
    newton_iters: int = 0
    wall_ms: float = 0.0

    @property
    def n(self) -> int:
        return len(self.psi)


def _arrays(f: FrameRecord):
    n = f.n
    shapes = {"x": (n, 3), "v": (n, 3), "psi": (n,), "vol": (n,), "ksur": (n,), "phase": (n,)}
    for k, shp in shapes.items():
        a = np.asarray(getattr(f, k), dtype="<f8")
        if a.shape != shp:
            raise FrameError(f"{k}: shape {a.shape}, expected {shp}")
        yield np.ascontiguousarray(a)


def encode_frame(f: FrameRecord) -> bytes:
    body = _HEAD.pack(MAGIC, VERSION, f.n, int(f.step), float(f.time))
    body += b"".join(a.tobytes() for a in _arrays(f))
    body += _FOOT.pack(float(f.worst_rel_error), int(f.newton_iters), float(f.wall_ms))
    return body + struct.pack("<I", zlib.crc32(body) & 0xFFFFFFFF)


def decode_frame(buf: bytes) -> FrameRecord:
    if len(buf) < _HEAD.size + _FOOT.size + 4:
        raise CrcError("truncated frame")
    magic, ver, n, step, time = _HEAD.unpack_from(buf, 0)
    if magic != MAGIC:
        raise FrameError(f"bad magic {magic!r}")
    if ver != VERSION:
        raise FrameError(f"unsupported frame version {ver}")
    need = _HEAD.size + 8 * 10 * n + _FOOT.size + 4
    if len(buf) != need:
        raise CrcError(f"frame size {len(buf)} != {need} (truncated or padded)")
    (crc,) = struct.unpack_from("<I", buf, len(buf) - 4)
    if zlib.crc32(buf[:-4]) & 0xFFFFFFFF != crc:
        raise CrcError("CRC32 mismatch")
    off = _HEAD.size
    out = {}
    for k, cnt in (("x", 3 * n), ("v", 3 * n), ("psi", n), ("vol", n), ("ksur", n), ("phase", n)):
        a = np.frombuffer(buf, dtype="<f8", count=cnt, offset=off).astype(np.float64)
        out[k] = a.reshape(n, 3) if cnt == 3 * n else a
        off += 8 * cnt
    w, it, ms = _FOOT.unpack_from(buf, off)
    return FrameRecord(step=step, time=time, worst_rel_error=w, newton_iters=it, wall_ms=ms, **out)


def write_frame(path: str, f: FrameRecord) -> None:
    with open(path, "wb") as fh:
        fh.write(encode_frame(f))


def read_frame(path: str) -> FrameRecord:
    with open(path, "rb") as fh:
        return decode_frame(fh.read())


def frame_from_state(state, diag: dict | None = None, wall_ms: float = 0.0, smf: int = 32) -> FrameRecord:
    """Snapshot of a fluid.FluidState after a step (volumes / free-surface areas
    of the step's final evaluation)."""
    from . import solver

    n = state.x.shape[0]
    vol, ksur = solver.last_state(n, smf)[:2]
    psi = state.psi if state.psi is not None else np.zeros(n)
    phase = getattr(state, "phase", None)
    return FrameRecord(step=state.step_index, time=state.time, x=state.x.cpu().numpy(), v=state.v.cpu().numpy(),
                       psi=psi.cpu().numpy() if hasattr(psi, "cpu") else np.asarray(psi),
                       vol=vol.cpu().numpy(), ksur=ksur.cpu().numpy(),
                       phase=np.zeros(n) if phase is None else np.asarray(phase, dtype=np.float64),
                       worst_rel_error=float((diag or {}).get("worst_final", 0.0)),
                       newton_iters=int((diag or {}).get("iterations", 0)), wall_ms=wall_ms)


def state_from_frame(f: FrameRecord, nu, rho):
    """Warm start: a fluid.FluidState carrying the frame's positions, velocities and weights."""
    import torch

    from . import fluid

    st = fluid.make_state(f.x, f.v, nu, rho)
    st.psi = torch.as_tensor(f.psi, dtype=torch.float64, device="cuda")
    st.step_index, st.time = int(f.step), float(f.time)
    return st
