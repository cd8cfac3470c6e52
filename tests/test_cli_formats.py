"""§8(f)-3 on the CPU: the pactrec driver's host paths and the file formats,
pinned to the reference compiled in oracle/_ref.

* PGRID / SIGSET / SIRN (io.hpp, nfield.hpp:235-289): files written by the
  reference read back bit-identically through the drop-in and are re-written
  byte-identically; error messages for truncated / bad-magic / non-finite /
  invalid files equal the reference's.
* generate_phantom + builtin specs (phantom.hpp:145-266) through
  `pactrec phantom`: the written rasters equal the reference's fp64 rasters
  rounded to f32, bit for bit (seeded jitter included).
* psf_from_transfer (aberration.hpp:407-445, GPU test): values within 1e-12,
  the same validation / numerical errors.
* the CLI contract of pactrec.cpp: subcommand tree, flag > PACT_* env >
  --config > default precedence, the resolved_config.ini echo (which loads
  back through --config to the same configuration), exit code 2 for bad
  arguments / specs, JSON phantom specs.
"""
import os
import shutil
import struct

import numpy as np
import pytest

import cli_helpers as H

REF = H.ref_io()
needs_ref = pytest.mark.skipif(REF is None, reason="oracle/_ref not built")


@pytest.fixture(scope="module", autouse=True)
def _built():
    H.build()


# ---- formats -------------------------------------------------------------------

@needs_ref
def test_pgrid_reference_written_roundtrip(tmp_path):
    rng = np.random.default_rng(0)
    v = rng.standard_normal((7, 11)) * 1e3
    a, b = str(tmp_path / "a.pgrid"), str(tmp_path / "b.pgrid")
    REF.write_pgrid(a, v, 0.125, -0.625, 3.5)
    rc, msg = H.io_tool(["pgrid", a, b])
    assert rc == 0, msg
    assert open(a, "rb").read() == open(b, "rb").read()
    got, geo = H.read_pgrid(b)
    assert geo == (0.125, -0.625, 3.5)
    np.testing.assert_array_equal(got, v.astype(np.float32))
    rc, (rv, rgeo) = REF.read_pgrid(b)
    assert rc == 0 and rgeo == geo
    np.testing.assert_array_equal(rv, v.astype(np.float32).astype(np.float64))


@needs_ref
def test_sigset_reference_written_roundtrip(tmp_path):
    rng = np.random.default_rng(1)
    d = rng.standard_normal((5, 33))
    meta = (25e-9, 1.3e-5, 40.0, 0.1, 1498.5)
    a, b = str(tmp_path / "a.sigset"), str(tmp_path / "b.sigset")
    REF.write_sigset(a, d, meta)
    rc, msg = H.io_tool(["sigset", a, b])
    assert rc == 0, msg
    assert open(a, "rb").read() == open(b, "rb").read()
    got, m = H.read_sigset(b)
    assert m == meta
    np.testing.assert_array_equal(got, d.astype(np.float32))


@needs_ref
def test_sirn_reference_written_roundtrip(tmp_path):
    rng = np.random.default_rng(2)
    hidden, layers = 16, 3
    n = hidden * 2 + hidden + (layers - 1) * (hidden * hidden + hidden) + hidden + 1
    theta = rng.standard_normal(n)
    a, b = str(tmp_path / "a.sirn"), str(tmp_path / "b.sirn")
    REF.write_sirn(a, hidden, layers, 30.0, 100.0, 1500.0, theta)
    rc, msg = H.io_tool(["sirn", a, b])
    assert rc == 0, msg
    assert open(a, "rb").read() == open(b, "rb").read()
    shapes, scal, t = H.read_sirn(b)
    assert shapes == [(16, 2), (16, 16), (16, 16), (1, 16)] and scal == (30.0, 100.0, 1500.0)
    np.testing.assert_array_equal(t, theta.astype(np.float32))
    rc, (shape, rscal, rt) = REF.load_sirn(b)
    assert rc == 0 and shape == (2, 16, 3)
    np.testing.assert_array_equal(rt, theta.astype(np.float32).astype(np.float64))


def _corrupt_cases(tmp_path):
    """(kind, file bytes) pairs covering every error path of the readers."""
    good_pg = b"PGRD" + struct.pack("<IIddd", 3, 2, 0.5, 0.0, 0.0) + np.arange(6, dtype="<f4").tobytes()
    nan_pg = bytearray(good_pg)
    nan_pg[36 + 8:36 + 12] = np.array([np.nan], "<f4").tobytes()
    cases = [
        ("pgrid", b""),
        ("pgrid", b"PGRX" + good_pg[4:]),
        ("pgrid", good_pg[:10]),            # inside height
        ("pgrid", good_pg[:30]),            # inside origin_y
        ("pgrid", good_pg[:-3]),            # last value cut
        ("pgrid", bytes(nan_pg)),           # non-finite value
        ("pgrid", b"PGRD" + struct.pack("<IIddd", 0, 2, 0.5, 0, 0)),
        ("pgrid", b"PGRD" + struct.pack("<IIddd", 2, 2, -1.0, 0, 0) + bytes(16)),
        ("pgrid", good_pg + b"trailing bytes are ignored"),
    ]
    sig_hdr = b"SIGS" + struct.pack("<II", 4, 3) + struct.pack("<ddddd", 1e-8, 0.0, 30.0, 0.0, 1500.0)
    sig = sig_hdr + np.ones(12, "<f4").tobytes()
    cases += [
        ("sigset", sig),
        ("sigset", sig[:20]),
        ("sigset", sig[:-1]),
        ("sigset", b"SIGS" + struct.pack("<II", 4, 3) + struct.pack("<ddddd", 1e-8, 0, 30, 0, 0.0)),
        ("sigset", b"SIGS" + struct.pack("<II", 2, 3) + struct.pack("<ddddd", 1e-8, 0, 30, 0, 1500)
         + np.ones(6, "<f4").tobytes()),                 # < 3 transducers
        ("sigset", b"SIGS" + struct.pack("<II", 4, 1) + struct.pack("<ddddd", 1e-8, 0, 30, 0, 1500)
         + np.ones(4, "<f4").tobytes()),                 # < 2 samples
        ("sigset", sig_hdr + np.array([1, 2, np.inf] + [0] * 9, "<f4").tobytes()),
    ]
    return cases


@needs_ref
def test_reader_errors_match_reference(tmp_path):
    for k, (kind, data) in enumerate(_corrupt_cases(tmp_path)):
        p = str(tmp_path / f"c{k}.{kind}")
        with open(p, "wb") as f:
            f.write(data)
        rc_ours, msg = H.io_tool([kind, p, str(tmp_path / f"o{k}")])
        rc_ref, ref_out = REF.read_pgrid(p) if kind == "pgrid" else REF.read_sigset(p)
        if rc_ref == 0:
            assert rc_ours == 0, (k, msg)
        else:
            assert rc_ours == rc_ref == 2, (k, rc_ours, rc_ref, msg)
            assert msg == "error: " + ref_out, (k, msg, ref_out)
    rc, msg = H.io_tool(["pgrid", str(tmp_path / "missing.pgrid"), str(tmp_path / "x")])
    assert rc == 2 and msg == f"error: cannot open for reading: {tmp_path}/missing.pgrid"


@needs_ref
def test_sirn_errors_match_reference(tmp_path):
    def sirn(shapes, scal=(30.0, 100.0, 1500.0), n=None, theta_val=0.5):
        n = sum(r * c + r for r, c in shapes) if n is None else n
        return (b"SIRN" + struct.pack("<I", len(shapes)) +
                b"".join(struct.pack("<II", r, c) for r, c in shapes) + struct.pack("<ddd", *scal) +
                np.full(n, theta_val, "<f4").tobytes())
    ok = [(8, 2), (8, 8), (1, 8)]
    cases = [sirn(ok), sirn([(8, 2)]), sirn(ok[:1] + [(8, 7), (1, 8)]), sirn(ok[:2] + [(2, 8)]),
             sirn(ok, scal=(0.0, 100.0, 1500.0)), sirn(ok, n=10), sirn(ok, theta_val=np.nan),
             sirn(ok)[:9]]
    for k, data in enumerate(cases):
        p = str(tmp_path / f"s{k}.sirn")
        with open(p, "wb") as f:
            f.write(data)
        rc_ours, msg = H.io_tool(["sirn", p, str(tmp_path / f"o{k}.sirn")])
        rc_ref, out = REF.load_sirn(p)
        assert rc_ours == rc_ref, (k, rc_ours, rc_ref, msg)
        if rc_ref:
            assert msg == "error: " + out, (k, msg, out)


# ---- psf_from_transfer ---------------------------------------------------------

@needs_ref
@pytest.mark.gpu  # psf_from_transfer runs on the device (pact_psf_from_transfer, fp64)
@pytest.mark.parametrize("P", [16, 12, 64])
def test_psf_from_transfer_matches_reference(tmp_path, P):
    rng = np.random.default_rng(P)
    psf = rng.standard_normal((P, P))
    spec = np.fft.fft2(psf)  # conjugate-symmetric by construction
    f_in, f_out = str(tmp_path / "s.f64"), str(tmp_path / "o.f64")
    np.stack([spec.real, spec.imag], -1).astype("<f8").tofile(f_in)
    rc, origin = H.io_tool(["psf", str(P), "0.1", f_in, f_out])
    assert rc == 0, origin
    ours = np.fromfile(f_out, "<f8").reshape(P, P)
    rc, ref = REF.psf_from_transfer(spec, P, 0.1)
    assert rc == 0
    np.testing.assert_allclose(ours, ref, rtol=0, atol=1e-12 * np.abs(ref).max())
    assert [float(x) for x in origin.split()] == pytest.approx([-(P // 2) * 0.1] * 2)
    # the zero-lag tap sits at (P/2, P/2)
    np.testing.assert_allclose(ours[P // 2, P // 2], psf[0, 0], atol=1e-12)
    # asymmetric spectrum: same ValidationError text
    bad = spec.copy()
    bad[1, 2] += 1e-3j
    np.stack([bad.real, bad.imag], -1).astype("<f8").tofile(f_in)
    rc, msg = H.io_tool(["psf", str(P), "0.1", f_in, f_out])
    rc_ref, ref_msg = REF.psf_from_transfer(bad, P, 0.1)
    assert rc == rc_ref == 2 and msg == "error: " + ref_msg


# ---- pactrec phantom (generate_phantom) ---------------------------------------

@needs_ref
@pytest.mark.parametrize("spec,seed,W,pitch", [("default", 0, 96, 0.25), ("default", 11, 64, 0.35),
                                              ("twobody", 0, 80, 0.25), ("empty", 3, 32, 0.5)])
def test_phantom_matches_reference(tmp_path, spec, seed, W, pitch):
    out = str(tmp_path / "o")
    rc, so, se = H.run(["phantom", "--spec", spec, "--seed", str(seed), "--grid-size", str(W),
                        "--pitch", str(pitch), "--out", out], tmp_path)
    assert rc == 0, se
    bg = REF.water_sos(26.0)
    pr_ref, sos_ref = REF.generate_phantom(spec, W, pitch, bg, (0.0, 0.0, 10.0), seed)
    pr, geo = H.read_pgrid(os.path.join(out, "pressure.pgrid"))
    so_, _ = H.read_pgrid(os.path.join(out, "sos.pgrid"))
    mk, _ = H.read_pgrid(os.path.join(out, "mask.pgrid"))
    np.testing.assert_array_equal(pr, pr_ref.astype(np.float32))
    np.testing.assert_array_equal(so_, sos_ref.astype(np.float32))
    assert geo == (pitch, -0.5 * (W - 1) * pitch, -0.5 * (W - 1) * pitch)
    xs = geo[1] + np.arange(W) * pitch
    X, Y = np.meshgrid(xs, xs)
    np.testing.assert_array_equal(mk, (np.hypot(X, Y) <= 10.0).astype(np.float32))
    if spec != "empty":
        assert pr.max() > 0 and (so_ != np.float32(bg)).any()


@needs_ref
def test_phantom_json_spec_equals_builtin(tmp_path):
    """A JSON file spelling out the builtin "twobody" spec gives the same rasters."""
    js = tmp_path / "twobody.json"
    js.write_text("""{"discs": [{"center": [0, 0], "radius": 9.0, "sos": 1561.0, "pressure": 0.05}],
                     "rings": [{"center": [0.0, 0.0], "radius": 9.0, "width": 0.25, "pressure": 0.8}],
                     "points": [{"pos": [0, 0], "amplitude": 1.5}, {"pos": [4.5, 1.0], "amplitude": 1.5},
                                {"pos": [-3.0, -4.0], "amplitude": 1.5}]}""")
    for name, spec in (("a", str(js)), ("b", "twobody")):
        rc, _, se = H.run(["phantom", "--spec", spec, "--grid-size", "72", "--pitch", "0.3",
                           "--out", str(tmp_path / name)], tmp_path)
        assert rc == 0, se
    for f in ("pressure.pgrid", "sos.pgrid", "mask.pgrid"):
        assert (tmp_path / "a" / f).read_bytes() == (tmp_path / "b" / f).read_bytes()


@pytest.mark.parametrize("text,needle", [
    ('{"discs": [{"center": [0, 0], "radius": 2, "colour": 1}]}', "unknown key 'colour' in disc"),
    ('{"bogus": 1}', "unknown key 'bogus' in top level"),
    ('{"discs": [{"center": [0, 0, 1], "radius": 2}]}', "disc.center must be [x, y]"),
    ('{"discs": [{"center": [0, 0]}]}', "missing key 'radius'"),
    ('{"discs": [', "bad JSON in"),
    ('{"discs": [{"center": [0, 0], "radius": 20}]}', "disc region extends outside the mask"),
    ('{"background_sos": 900}', "background SOS outside [1300, 1800] m/s"),
])
def test_phantom_bad_specs_exit_2(tmp_path, text, needle):
    js = tmp_path / "s.json"
    js.write_text(text)
    rc, _, se = H.run(["phantom", "--spec", str(js), "--grid-size", "16", "--out",
                       str(tmp_path / "o")], tmp_path)
    assert rc == 2 and needle in se, se


# ---- the CLI contract ------------------------------------------------------------

def _resolved(d):
    out = {}
    section = ""
    for line in open(os.path.join(d, "resolved_config.ini")):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        if line.startswith("["):
            section = line[1:-1]
            continue
        k, v = line.split("=", 1)
        out[(section, k)] = v.strip('"')
    return out


def test_cli_tree_and_parse_errors(tmp_path):
    rc, so, _ = H.run(["--help"], tmp_path)
    assert rc == 0 and all(s in so for s in ("phantom", "simulate", "recon", "psf", "eval"))
    rc, so, _ = H.run(["recon", "nf", "--help"], tmp_path)
    assert rc == 0 and "--implicit-grad,--no-implicit-grad" in so and "PACT_STEPS_PER_EPOCH" in so
    for args in ([], ["recon"], ["psf"], ["bogus"], ["phantom", "--nope", "1"],
                 ["phantom", "--grid-size", "abc"], ["phantom", "--grid-size"],
                 ["recon", "das", "--spreading"]):
        rc, _, se = H.run(args, tmp_path)
        assert rc == 2, (args, se)


def test_cli_precedence_flag_env_config_default(tmp_path):
    cfg = tmp_path / "c.ini"
    cfg.write_text("# comment\n[phantom]\ngrid-size=24\nseed=7\npitch = 0.4\nspec=\"empty\"\n")
    out = tmp_path / "o"
    rc, _, se = H.run(["--config", str(cfg), "phantom", "--pitch", "0.5", "--out", str(out)],
                      tmp_path, env={"PACT_SEED": "3", "PACT_PITCH": "0.45"})
    assert rc == 0, se
    r = _resolved(out)
    assert r[("phantom", "grid-size")] == "24"   # config
    assert r[("phantom", "seed")] == "3"         # env beats config
    assert r[("phantom", "pitch")] == "0.5"      # flag beats env and config
    assert r[("phantom", "spec")] == "empty"     # config
    assert r[("phantom", "mask-radius")] == "10"  # default
    _, geo = H.read_pgrid(str(out / "sos.pgrid"))
    assert geo[0] == 0.5
    # the echo loads back through --config to the same configuration
    out2 = tmp_path / "o2"
    rc, _, se = H.run(["--config", str(out / "resolved_config.ini"), "phantom", "--out", str(out2)],
                      tmp_path)
    assert rc == 0, se
    r2 = _resolved(out2)
    r2[("phantom", "out")] = r[("phantom", "out")]
    assert r2 == r
    # flat (unsectioned) keys of the selected command, dotted keys, unknown keys
    flat = tmp_path / "flat.ini"
    flat.write_text("grid-size=20\nphantom.seed=5\n")
    rc, _, se = H.run(["--config", str(flat), "phantom", "--out", str(tmp_path / "o3")], tmp_path)
    assert rc == 0, se
    r3 = _resolved(tmp_path / "o3")
    assert r3[("phantom", "grid-size")] == "20" and r3[("phantom", "seed")] == "5"
    bad = tmp_path / "bad.ini"
    bad.write_text("[phantom]\nno-such-option=1\n")
    rc, _, se = H.run(["--config", str(bad), "phantom", "--out", str(tmp_path / "o4")], tmp_path)
    assert rc == 2
    # another subcommand's section is accepted and ignored
    other = tmp_path / "other.ini"
    other.write_text("[recon.das]\ngrid-size=99\n[phantom]\ngrid-size=18\n")
    rc, _, se = H.run(["--config", str(other), "phantom", "--out", str(tmp_path / "o5")], tmp_path)
    assert rc == 0, se
    assert _resolved(tmp_path / "o5")[("phantom", "grid-size")] == "18"


def test_cli_flags_and_vectors_parse(tmp_path):
    """--no-flag / --flag=value and vector options resolve as CLI11 does (checked on the
    resolved echo of commands that then fail on a missing input file: exit 2)."""
    out = tmp_path / "o"
    rc, _, se = H.run(["simulate", "--no-spreading", "--pressure", "nope.pgrid", "--out", str(out)],
                      tmp_path)
    assert rc == 2 and "cannot open for reading: nope.pgrid" in se
    assert _resolved(out)[("simulate", "spreading")] == "false"
    rc, _, se = H.run(["psf", "dump", "--index", "3", "1", "--n-angles=64", "--sos", "nope.pgrid",
                       "--out", str(out)], tmp_path, env={"PACT_DELAYS": "-1:1:3"})
    assert rc == 2
    r = _resolved(out)
    assert r[("psf.dump", "index")] == "3 1" and r[("psf.dump", "n-angles")] == "64"
    assert r[("psf.dump", "delays")] == "-1:1:3"
    rc, _, _ = H.run(["psf", "dump", "--sos", "x", "--out", str(out)], tmp_path,
                     env={"PACT_INDEX": "4,5"})
    assert _resolved(out)[("psf.dump", "index")] == "4 5"


@needs_ref
def test_simulate_window_matches_reference(tmp_path):
    """pact_simulate_window (host): the automatic acquisition window of
    simulate_signals (phantom.hpp:293-334) equals the reference's, and an
    explicit window that misses the arrivals fails with its message."""
    import math

    from paper_2409_10876_b200.api import GridSpec, RingGeometry, check, simulate_window
    from paper_2409_10876_b200 import _abi
    bg = REF.water_sos(20.0)
    pr, so = REF.generate_phantom("default", 48, 0.4, bg, (0.0, 0.0, 10.0), 2)
    grid = GridSpec.centered(48, 48, 0.4)
    for ring, sigma, dt in (((64, 30.0, 0.0), 100e-9, 25e-9), ((32, 22.0, 0.3), 60e-9, 20e-9)):
        t0, T, _ = REF.simulate(pr, so, (0.4, grid.origin_x, grid.origin_y), (0.0, 0.0, 10.0), bg,
                                ring, sigma, dt, False, 0.05)
        m = simulate_window(grid, pr, so, bg, RingGeometry(*ring), sigma, dt)
        assert (m.t0, m.n_samples, m.dt, m.background_sos) == (t0, T, dt, bg)
    with pytest.raises(_abi.ValidationError, match="time window too short"):
        simulate_window(grid, pr, so, bg, RingGeometry(64, 30.0), 100e-9, 25e-9, 0.0, 10)
    with pytest.raises(_abi.ValidationError, match="pressure-bearing pixel outside"):
        simulate_window(grid, pr, so, bg, RingGeometry(64, 5.0), 100e-9, 25e-9)
    assert math.isfinite(m.t0)
