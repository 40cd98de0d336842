"""Router-bank wire format: byte compatibility with the
reference's save_bank / load_bank and its corruption checks, mirroring
pkg/tests/test_calibration.py:366-457 (TestBankSerialization).

tests/golden/ref.bank was written by the real reference
(tests/golden/make_bank_golden.py)."""

import os
import struct
import zlib

import numpy as np
import pytest

from tests.conftest import GOLDEN

import paper_2603_21365_b200 as P
from paper_2603_21365_b200 import bank_io as B

REF_BANK = os.path.join(GOLDEN, "ref.bank")


@pytest.fixture()
def bank():
    g = np.random.Generator(np.random.PCG64(99))
    routers = {k: ((g.standard_normal((16, 48)) * 0.2).astype(np.float32),
                   (g.standard_normal((1, 16)) * 0.2).astype(np.float32)) for k in (3, 7, 11)}
    return P.make_bank(routers, num_layers=12, tau=0.97, model_digest=42)


def test_reference_file_loads_field_by_field():
    bk = B.load_bank(REF_BANK)
    assert (bk.hidden_dim, bk.bottleneck, bk.interval, bk.num_layers) == (64, 32, 4, 12)
    assert bk.tau == pytest.approx(0.98) and bk.eps == pytest.approx(1e-6)
    assert bk.model_digest == 0x0123456789ABCDEF
    assert bk.checkpoints == (3, 7, 11)
    g = np.random.Generator(np.random.PCG64(515))  # make_bank_golden.py's stream
    for i, k in enumerate((3, 7, 11)):
        w_down = (g.standard_normal((32, 64)) * 0.1).astype(np.float32)
        w_up = (g.standard_normal((1, 32)) * 0.1).astype(np.float32)
        assert np.array_equal(bk.routers[k].w_down, w_down)
        assert np.array_equal(bk.routers[k].w_up, w_up)
        st = bk.stats[k]
        assert (st.examples, st.positives, st.flags) == (1000 + i, 100 * i, i & 1)
        assert st.final_loss == pytest.approx(0.25 + i) and st.accuracy == pytest.approx(0.5 + 0.125 * i)


def test_reference_file_resaves_bitwise(tmp_path):
    out = tmp_path / "again.bank"
    B.save_bank(B.load_bank(REF_BANK), out)
    assert out.read_bytes() == open(REF_BANK, "rb").read()


def test_round_trip_and_size_formula(bank, tmp_path):
    path = tmp_path / "routers.bank"
    B.save_bank(bank, path)
    assert path.stat().st_size == B.bank_file_size(48, 16, 3)
    loaded = B.load_bank(path)
    assert loaded.checkpoints == bank.checkpoints and loaded.model_digest == 42
    for k in bank.checkpoints:
        assert np.array_equal(loaded.routers[k].w_down, bank.routers[k].w_down)
        assert np.array_equal(loaded.routers[k].w_up, bank.routers[k].w_up)
    p2 = tmp_path / "b.bank"
    B.save_bank(loaded, p2)
    assert p2.read_bytes() == path.read_bytes()


def test_truncation_mid_weights(bank, tmp_path):
    path = tmp_path / "cut.bank"
    B.save_bank(bank, path)
    path.write_bytes(path.read_bytes()[:-100])
    with pytest.raises(B.TruncatedError):
        B.load_bank(path)


def test_flipped_byte_fails_checksum(bank, tmp_path):
    path = tmp_path / "flip.bank"
    B.save_bank(bank, path)
    data = bytearray(path.read_bytes())
    data[60] ^= 0x01
    path.write_bytes(bytes(data))
    with pytest.raises(B.ChecksumError):
        B.load_bank(path)


def test_bad_magic(bank, tmp_path):
    path = tmp_path / "magic.bank"
    B.save_bank(bank, path)
    data = bytearray(path.read_bytes())
    data[:4] = b"EDIT"
    path.write_bytes(bytes(data))
    with pytest.raises(B.BadMagicError):
        B.load_bank(path)


def _container(fields: bytes) -> bytes:
    body = b"TIDE" + fields
    return body + struct.pack("<I", zlib.crc32(body) & 0xFFFFFFFF)


def test_unknown_version(tmp_path):
    path = tmp_path / "future.bank"
    path.write_bytes(_container(struct.pack("<I", 99)))
    with pytest.raises(B.VersionError):
        B.load_bank(path)


def test_implausible_metadata(tmp_path):
    path = tmp_path / "dims.bank"
    path.write_bytes(_container(struct.pack("<IIIIffIIQ", 1, 0, 4, 4, 0.98, 1e-6, 12, 1, 0)))
    with pytest.raises(B.DimensionError):
        B.load_bank(path)


def test_trailing_garbage_detected(bank, tmp_path):
    path = tmp_path / "extra.bank"
    B.save_bank(bank, path)
    path.write_bytes(path.read_bytes() + b"\x00" * 16)
    with pytest.raises(B.DimensionError, match="trailing"):
        B.load_bank(path)


def test_tiny_file_is_truncation(tmp_path):
    path = tmp_path / "tiny.bank"
    path.write_bytes(b"TID")
    with pytest.raises(B.TruncatedError):
        B.load_bank(path)


def test_errors_share_base_class():
    for cls in (B.BadMagicError, B.VersionError, B.TruncatedError, B.ChecksumError,
                B.DimensionError):
        assert issubclass(cls, B.BinaryFormatError)


@pytest.mark.gpu
def test_load_to_device_installs_router_weights():
    from tests.gpu_helpers import need_gpu
    need_gpu()
    import torch
    from paper_2603_21365_b200 import _native as N
    from paper_2603_21365_b200 import router_ops as R
    bk = B.load_bank(REF_BANK, device="cuda", dtype=torch.bfloat16)
    ref = B.load_bank(REF_BANK)
    for k in bk.checkpoints:
        wd, wu = R.device_weights(bk.routers[k], N.BF16, torch.device("cuda"))
        want = torch.from_numpy(ref.routers[k].w_down).to(torch.bfloat16)
        assert torch.equal(wd.cpu(), want)
        assert torch.equal(wu.cpu(), torch.from_numpy(ref.routers[k].w_up.reshape(-1)))
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    h = torch.randn((300, 64), generator=g, device="cuda").to(torch.bfloat16)
    s1 = P.fused_layernorm_route(h, bk.routers[7])
    s2 = P.fused_layernorm_route(h, ref.routers[7])
    assert torch.equal(s1, s2)
