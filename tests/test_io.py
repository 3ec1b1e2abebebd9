"""MOMV binary ingest: format parity with the reference and device upload."""

import struct

import numpy as np
import pytest

import paper_1911_03813_b200 as mcp
from oracle import momentcp_oracle as om


def _write(path, V):
    mcp.write_observations_binary(str(path), mcp.ObservationSet(V))


def test_round_trip_host_view(tmp_path):
    V = np.random.default_rng(0).standard_normal((5, 9))
    _write(tmp_path / "a.momv", V)
    obs = mcp.read_observations_binary(str(tmp_path / "a.momv"))
    assert obs.n == 5 and obs.p == 9 and np.array_equal(obs.V, V)
    shard = mcp.read_observations_binary(str(tmp_path / "a.momv"), rows=(3, 7))
    assert shard.p == 4 and np.array_equal(shard.V, V[:, 3:7])
    assert np.allclose(shard.weights(), 1.0 / 9)          # a shard keeps 1/p of the file


def test_header_errors(tmp_path):
    V = np.ones((2, 3))
    _write(tmp_path / "ok.momv", V)
    raw = (tmp_path / "ok.momv").read_bytes()
    (tmp_path / "magic.momv").write_bytes(b"XXXX" + raw[4:])
    (tmp_path / "ver.momv").write_bytes(raw[:4] + struct.pack("<I", 2) + raw[8:])
    (tmp_path / "short.momv").write_bytes(raw[:-8])
    (tmp_path / "hdr.momv").write_bytes(raw[:10])
    for name in ("magic", "ver", "short", "hdr"):
        with pytest.raises(mcp.ParseError):
            mcp.read_observations_binary(str(tmp_path / f"{name}.momv"))


def test_written_file_matches_reference_layout(tmp_path):
    V = np.arange(6, dtype=float).reshape(2, 3)
    _write(tmp_path / "l.momv", V)
    raw = (tmp_path / "l.momv").read_bytes()
    assert raw[:4] == b"MOMV" and struct.unpack("<IQQ", raw[4:24]) == (1, 2, 3)
    assert np.array_equal(np.frombuffer(raw[24:], "<f8"), V.ravel(order="F"))


@pytest.mark.gpu
def test_ingested_set_evaluates_like_the_original(tmp_path):
    rng = np.random.default_rng(4)
    V = rng.standard_normal((20, 5000))
    _write(tmp_path / "v.momv", V)
    lam, A = rng.standard_normal(5), rng.standard_normal((20, 5))
    a = mcp.fg_implicit(mcp.read_observations_binary(str(tmp_path / "v.momv")), lam, A, 3)
    b = mcp.fg_implicit(mcp.ObservationSet(V), lam, A, 3)
    assert a.f == b.f and np.array_equal(a.g_A, b.g_A)
    Vbad = V.copy()
    Vbad[3, 17] = np.nan
    _write(tmp_path / "bad.momv", np.nan_to_num(Vbad))
    raw = bytearray((tmp_path / "bad.momv").read_bytes())
    raw[24 + 8 * (17 * 20 + 3): 24 + 8 * (17 * 20 + 4)] = struct.pack("<d", float("nan"))
    (tmp_path / "bad.momv").write_bytes(bytes(raw))
    with pytest.raises(ValueError):
        mcp.fg_implicit(mcp.read_observations_binary(str(tmp_path / "bad.momv")), lam, A, 3)
    # shard partials sum to the full evaluation
    nu = np.full(5000, 1 / 5000)
    f, gl, gA = om.fg_implicit(V, nu, lam, A, 3)
    assert abs(a.f - f) <= 1e-12 * max(1, abs(f))
