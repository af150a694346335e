"""CPU: FLOP v1 checkpoints are byte-identical with the reference's writer
and readable by it, and the loader rejects what the reference rejects
(pkg/tests/test_checkpoint.py:39-206)."""

from __future__ import annotations

import os
import struct

import numpy as np
import pytest

import helpers as H
import refbridge as R
from devstate import bits

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _host(st: dict, t: int):
    from paper_2602_23349_b200.host import HostFlashState

    return HostFlashState(st["weights.lp"], st["weights.rho"], st["momentum.codes"], st["momentum.scales"],
                          st.get("variance.codes"), st.get("variance.scales"), t)


def _same(a, b):
    for k in ("lp", "rho", "m_codes", "m_scales", "v_codes", "v_scales"):
        x, y = getattr(a, k), getattr(b, k)
        assert (x is None) == (y is None), k
        if x is not None:
            assert np.array_equal(bits(x), bits(y)), k
    assert a.t == b.t


@pytest.mark.parametrize("opt,n", [("adamw", 1003), ("sgd", 64), ("lion", 33)])
def test_golden_reference_files_roundtrip_bytes(opt, n, tmp_path):
    """Load a file the reference wrote, write it back: identical bytes."""
    from paper_2602_23349_b200 import checkpoint as C

    src = os.path.join(GOLD, f"ckpt_{opt}.flop")
    hs = C.load_checkpoint(src)
    assert hs.length == n and C.inspect_checkpoint(src)["optimizer"] == opt
    out = tmp_path / "x.flop"
    nbytes = C.save_checkpoint(hs, out, optimizer=opt)
    assert open(src, "rb").read() == open(out, "rb").read()
    assert nbytes == os.path.getsize(src)


def test_int16_corrections_roundtrip(tmp_path):
    from paper_2602_23349_b200 import checkpoint as C

    src = os.path.join(GOLD, "ckpt_adamw_rho16.flop")
    hs = C.load_checkpoint(src)
    assert hs.rho.dtype == np.int16
    C.save_checkpoint(hs, tmp_path / "y.flop")
    assert open(src, "rb").read() == open(tmp_path / "y.flop", "rb").read()


@pytest.mark.parametrize("opt", ["adamw", "sgd", "lion"])
def test_random_roundtrip_and_u64_step(opt, tmp_path):
    from paper_2602_23349_b200 import checkpoint as C

    rng = np.random.default_rng(3)
    for i in range(10):
        n = int(rng.integers(1, 5000))
        hs = _host(H.random_state(rng, n, opt), int(rng.integers(0, 2**63)))
        p = tmp_path / f"{i}.flop"
        C.save_checkpoint(hs, p, optimizer=opt)
        _same(hs, C.load_checkpoint(p))


def test_payload_formula(tmp_path):
    """test_checkpoint.py:180-188: 2n + n + n + n + 2*(n/32)*2 for AdamW."""
    from paper_2602_23349_b200 import checkpoint as C

    n = 4096
    hs = _host(H.random_state(np.random.default_rng(0), n, "adamw"), 1)
    C.save_checkpoint(hs, tmp_path / "p.flop")
    assert C.payload_bytes(tmp_path / "p.flop")["payload_bytes"] == 2 * n + n + n + n + 2 * (n // 32) * 2


def test_lion_tag_inference_matches_reference(tmp_path):
    """checkpoint.py:128-131: without optimizer=, a Lion state is tagged sgd."""
    from paper_2602_23349_b200 import checkpoint as C

    hs = _host(H.random_state(np.random.default_rng(1), 64, "lion"), 1)
    C.save_checkpoint(hs, tmp_path / "l.flop")
    assert C.inspect_checkpoint(tmp_path / "l.flop")["optimizer"] == "sgd"


class TestCorruption:
    def _file(self, tmp_path):
        from paper_2602_23349_b200 import checkpoint as C

        hs = _host(H.random_state(np.random.default_rng(2), 256, "adamw"), 3)
        p = tmp_path / "c.flop"
        C.save_checkpoint(hs, p)
        return p, bytearray(open(p, "rb").read())

    def _expect(self, tmp_path, blob, match):
        from paper_2602_23349_b200 import checkpoint as C

        q = tmp_path / "bad.flop"
        open(q, "wb").write(bytes(blob))
        with pytest.raises(C.CheckpointError, match=match):
            C.load_checkpoint(q)

    @staticmethod
    def _recrc(blob):
        import zlib

        blob[-4:] = struct.pack("<I", zlib.crc32(bytes(blob[:-4])))
        return blob

    def test_crc(self, tmp_path):
        p, b = self._file(tmp_path)
        b[40] ^= 1
        self._expect(tmp_path, b, "crc-mismatch")

    def test_truncated(self, tmp_path):
        p, b = self._file(tmp_path)
        self._expect(tmp_path, b[:20], "truncated")
        self._expect(tmp_path, self._recrc(b[:-100]), "truncated")

    def test_magic_and_version(self, tmp_path):
        p, b = self._file(tmp_path)
        m = bytearray(b)
        m[0:4] = b"FLOQ"
        self._expect(tmp_path, self._recrc(m), "bad-magic")
        v = bytearray(b)
        v[4:6] = struct.pack("<H", 2)
        self._expect(tmp_path, self._recrc(v), "unsupported-version")

    def test_trailing_bytes(self, tmp_path):
        p, b = self._file(tmp_path)
        self._expect(tmp_path, self._recrc(b[:-4] + b"\0\0\0\0" + b"\0\0\0\0"), "trailing")

    def test_minus_128_rejected(self, tmp_path):
        from paper_2602_23349_b200 import checkpoint as C

        st = H.random_state(np.random.default_rng(4), 64, "adamw")
        st["weights.rho"][3] = -128
        C.save_checkpoint(_host(st, 1), tmp_path / "r.flop")
        with pytest.raises(C.CheckpointError, match="invalid-correction-code"):
            C.load_checkpoint(tmp_path / "r.flop")


@pytest.mark.skipif(not R.available(), reason="reference not importable here")
@pytest.mark.parametrize("opt", ["adamw", "sgd", "lion"])
def test_byte_identical_to_live_reference(opt, tmp_path):
    from paper_2602_23349_b200 import checkpoint as C

    fo = R.flashopt()
    rng = np.random.default_rng(11)
    for i in range(5):
        n = int(rng.integers(1, 3000))
        st = H.random_state(rng, n, opt)
        t = int(rng.integers(0, 2**40))
        fo.checkpoint.save_checkpoint(R.to_ref_state(st, t), tmp_path / "ref.flop", optimizer=opt)
        C.save_checkpoint(_host(st, t), tmp_path / "ours.flop", optimizer=opt)
        assert open(tmp_path / "ref.flop", "rb").read() == open(tmp_path / "ours.flop", "rb").read()
        back = fo.checkpoint.load_checkpoint(tmp_path / "ours.flop")
        assert np.array_equal(back.weights.lp_values, st["weights.lp"])
        assert np.array_equal(back.momentum.scales.view(np.uint16), st["momentum.scales"].view(np.uint16))
