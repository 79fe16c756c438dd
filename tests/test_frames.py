"""POTF frames (cli_io write_frame / read_frame): bit-exact round
trip, magic / version / CRC checks, truncation detected.  CPU only."""
import numpy as np
import pytest


def _frame(n=50, seed=0):
    from paper_2601_05765_b200.frames import FrameRecord

    r = np.random.default_rng(seed)
    return FrameRecord(step=7, time=0.007, x=r.random((n, 3)), v=r.normal(size=(n, 3)), psi=r.random(n) * 1e-4,
                       vol=r.random(n), ksur=r.random(n), phase=np.zeros(n), worst_rel_error=3e-3,
                       newton_iters=2, wall_ms=12.5)


def test_round_trip_bit_exact(tmp_path):
    from paper_2601_05765_b200 import frames

    f = _frame()
    p = tmp_path / "a.potf"
    frames.write_frame(str(p), f)
    g = frames.read_frame(str(p))
    for k in ("x", "v", "psi", "vol", "ksur", "phase"):
        assert np.array_equal(getattr(f, k), getattr(g, k)), k
    assert (g.step, g.time, g.worst_rel_error, g.newton_iters, g.wall_ms) == (7, 0.007, 3e-3, 2, 12.5)
    assert open(p, "rb").read(4) == b"POTF"


def test_corruption_and_truncation_detected():
    from paper_2601_05765_b200 import frames

    buf = bytearray(frames.encode_frame(_frame()))
    with pytest.raises(frames.CrcError):
        frames.decode_frame(bytes(buf[:-9]))
    bad = bytearray(buf)
    bad[100] ^= 1
    with pytest.raises(frames.CrcError):
        frames.decode_frame(bytes(bad))
    bad = bytearray(buf)
    bad[0:4] = b"XXXX"
    with pytest.raises(frames.FrameError):
        frames.decode_frame(bytes(bad))
