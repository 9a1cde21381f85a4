"""PFD1 field dumps (S/fielddump.py) byte-for-byte against dumps written by
the reference itself (tests/golden/backstep_u*.pfd, from a multi-block
backward-facing-step field), read-back and corruption checks; the GPU tier
dumps a device tensor."""

import os

import numpy as np
import pytest
import torch

from paper_2505_16992_b200 import fielddump, mesh

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _field():
    return np.load(os.path.join(GOLD, "backstep_u.npy"))


@pytest.mark.parametrize("precision,name", [("double", "backstep_u.pfd"),
                                            ("single",
                                             "backstep_u_single.pfd")])
def test_dump_matches_reference_bytes(tmp_path, precision, name):
    dom = mesh.make_backstep(2)
    out = tmp_path / "u.pfd"
    n = fielddump.dump_state(str(out), dom, _field(), time=1.25,
                             precision=precision)
    ref = open(os.path.join(GOLD, name), "rb").read()
    got = open(out, "rb").read()
    assert n == len(ref)
    assert got == ref
    # torch (host) input writes the same bytes
    fielddump.dump_state(str(out), dom, torch.as_tensor(_field()), time=1.25,
                         precision=precision)
    assert open(out, "rb").read() == ref


def test_read_back_and_errors(tmp_path):
    dom = mesh.make_backstep(2)
    arr, t, prec = fielddump.load_state(os.path.join(GOLD, "backstep_u.pfd"),
                                        dom)
    assert t == 1.25 and prec == "double"
    np.testing.assert_array_equal(arr, _field())
    arr32, _, prec32 = fielddump.load_state(
        os.path.join(GOLD, "backstep_u_single.pfd"), dom)
    assert prec32 == "single" and arr32.dtype == np.float32
    bad = bytearray(open(os.path.join(GOLD, "backstep_u.pfd"), "rb").read())
    bad[-10] ^= 0xFF
    p = tmp_path / "bad.pfd"
    p.write_bytes(bytes(bad))
    with pytest.raises(fielddump.DumpError):
        fielddump.read_fields(str(p))
    p.write_bytes(b"XXXX" + bytes(bad[4:]))
    with pytest.raises(fielddump.DumpError):
        fielddump.read_fields(str(p))
    with pytest.raises(fielddump.DumpError):
        fielddump.load_state(os.path.join(GOLD, "backstep_u.pfd"),
                             mesh.make_cavity((4, 4)))
    with pytest.raises(ValueError):
        fielddump.write_fields(str(p), [])


@pytest.mark.gpu
def test_dump_device_tensor(tmp_path):
    dom = mesh.make_backstep(2)
    u = torch.as_tensor(_field(), device="cuda:0")
    out = tmp_path / "u.pfd"
    fielddump.dump_state(str(out), dom, u, time=1.25)
    assert open(out, "rb").read() == open(os.path.join(GOLD,
                                                       "backstep_u.pfd"),
                                          "rb").read()
    back, _, _ = fielddump.load_state(str(out), dom, device="cuda:0")
    assert torch.equal(back, u)
