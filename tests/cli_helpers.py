"""Shared helpers of the §8(f)-3 tests (pactrec CLI, PGRID / SIGSET / SIRN).

* build(): make the pactrec binary and tests/cpp/io_tool (host-only drivers);
* run(): run pactrec in a scratch directory, returning (rc, stdout, stderr);
* numpy readers of the three formats (a third, independent decoder);
* RefIO: the reference's own io.hpp / nfield.hpp / phantom.hpp / psf_from_transfer
  compiled in oracle/_ref (libpact_ref.so) behind ctypes (test infrastructure).
"""
import ctypes as C
import os
import struct
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PACTREC = os.path.join(ROOT, "paper_2409_10876_b200", "bin", "pactrec")
IO_TOOL = os.path.join(ROOT, "build", "io_tool")
REF_PATH = os.path.join(ROOT, "oracle", "_ref", "libpact_ref.so")


def build():
    r = subprocess.run(["make", "-C", ROOT, "lib", "pactrec"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    os.makedirs(os.path.dirname(IO_TOOL), exist_ok=True)
    libdir = os.path.join(ROOT, "paper_2409_10876_b200", "lib")
    src = os.path.join(ROOT, "tests", "cpp", "io_tool.cpp")
    if not os.path.exists(IO_TOOL) or os.path.getmtime(IO_TOOL) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(libdir, "libpact_cuda.so"))):
        cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
               "-I", os.path.join(ROOT, "paper_2409_10876_b200", "include"), src, "-o", IO_TOOL,
               "-L", libdir, "-lpact_cuda", f"-Wl,-rpath,{libdir}"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-3000:]


def run(args, cwd, env=None, timeout=900):
    e = {k: v for k, v in os.environ.items() if not k.startswith("PACT_") or k == "PACT_DEVICE"}
    if env:
        e.update(env)
    r = subprocess.run([PACTREC] + list(args), cwd=cwd, env=e, capture_output=True, text=True,
                       timeout=timeout)
    return r.returncode, r.stdout, r.stderr


def io_tool(args):
    r = subprocess.run([IO_TOOL] + list(args), capture_output=True, text=True, timeout=120)
    return r.returncode, r.stdout.strip()


# ---- numpy decoders ----------------------------------------------------------

def read_pgrid(path):
    b = open(path, "rb").read()
    assert b[:4] == b"PGRD"
    w, h = struct.unpack_from("<II", b, 4)
    pitch, ox, oy = struct.unpack_from("<ddd", b, 12)
    v = np.frombuffer(b, "<f4", w * h, 36).reshape(h, w)
    return v, (pitch, ox, oy)


def write_pgrid(path, values, pitch, ox, oy):
    v = np.ascontiguousarray(values, "<f4")
    h, w = v.shape
    with open(path, "wb") as f:
        f.write(b"PGRD" + struct.pack("<IIddd", w, h, pitch, ox, oy) + v.tobytes())


def read_sigset(path):
    b = open(path, "rb").read()
    assert b[:4] == b"SIGS"
    n, t = struct.unpack_from("<II", b, 4)
    meta = struct.unpack_from("<ddddd", b, 12)  # dt, t0, radius, angle_offset, background_sos
    v = np.frombuffer(b, "<f4", n * t, 52).reshape(n, t)
    return v, meta


def read_sirn(path):
    b = open(path, "rb").read()
    assert b[:4] == b"SIRN"
    (nl,) = struct.unpack_from("<I", b, 4)
    shapes = [struct.unpack_from("<II", b, 8 + 8 * i) for i in range(nl)]
    o = 8 + 8 * nl
    scal = struct.unpack_from("<ddd", b, o)
    n = sum(r * c + r for r, c in shapes)
    theta = np.frombuffer(b, "<f4", n, o + 24)
    return shapes, scal, theta


# ---- the reference (oracle/_ref) ------------------------------------------------

_D, _I, _P = C.c_double, C.c_int, C.c_void_p


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class RefIO:
    def __init__(self):
        self.lib = C.CDLL(REF_PATH)
        L = self.lib
        L.ref_generate_phantom.argtypes = [C.c_char_p, _I, _I, _D, _D, _D, _D, _D, C.c_uint64, _P, _P]
        L.ref_read_pgrid.argtypes = [C.c_char_p, C.POINTER(_I), C.POINTER(_I), _P, _P, C.c_size_t]
        L.ref_write_pgrid.argtypes = [C.c_char_p, _I, _I, _D, _D, _D, _P]
        L.ref_read_sigset.argtypes = [C.c_char_p, C.POINTER(_I), C.POINTER(_I), _P, _P, C.c_size_t]
        L.ref_write_sigset.argtypes = [C.c_char_p, _I, _I, _P, _P]
        L.ref_load_sirn.argtypes = [C.c_char_p, _P, _P, _P, C.c_size_t]
        L.ref_write_sirn.argtypes = [C.c_char_p, _I, _I, _D, _D, _D, _P]
        L.ref_psf_from_transfer.argtypes = [_I, _D, _P, _P]
        L.ref_simulate_auto.argtypes = [_I, _I, _D, _D, _D, _P, _P, _D, _D, _D, _D, _I, _D, _D,
                                        _D, _D, _I, _D, _P, _P, C.c_size_t]
        L.ref_water_sos.argtypes = [_D]
        L.ref_water_sos.restype = _D
        L.ref_last_error.restype = C.c_char_p

    def err(self):
        return self.lib.ref_last_error().decode()

    def generate_phantom(self, name, W, pitch, bg, mask, seed):
        pr = np.zeros((W, W))
        so = np.zeros((W, W))
        rc = self.lib.ref_generate_phantom(name.encode(), W, W, pitch, bg, mask[0], mask[1],
                                           mask[2], seed, _p(pr), _p(so))
        assert rc == 0, self.err()
        return pr, so

    def read_pgrid(self, path):
        w, h = _I(), _I()
        geo = np.zeros(3)
        rc = self.lib.ref_read_pgrid(path.encode(), C.byref(w), C.byref(h), _p(geo), None, 0)
        if rc != 0:
            return rc, self.err()
        v = np.zeros((h.value, w.value))
        self.lib.ref_read_pgrid(path.encode(), C.byref(w), C.byref(h), _p(geo), _p(v), v.size)
        return 0, (v, tuple(geo))

    def write_pgrid(self, path, values, pitch, ox, oy):
        v = np.ascontiguousarray(values, np.float64)
        rc = self.lib.ref_write_pgrid(path.encode(), v.shape[1], v.shape[0], pitch, ox, oy, _p(v))
        assert rc == 0, self.err()

    def read_sigset(self, path):
        n, t = _I(), _I()
        meta = np.zeros(5)
        rc = self.lib.ref_read_sigset(path.encode(), C.byref(n), C.byref(t), _p(meta), None, 0)
        if rc != 0:
            return rc, self.err()
        v = np.zeros((n.value, t.value))
        self.lib.ref_read_sigset(path.encode(), C.byref(n), C.byref(t), _p(meta), _p(v), v.size)
        return 0, (v, tuple(meta))

    def write_sigset(self, path, data, meta):
        d = np.ascontiguousarray(data, np.float64)
        m = np.asarray(meta, np.float64)
        rc = self.lib.ref_write_sigset(path.encode(), d.shape[0], d.shape[1], _p(m), _p(d))
        assert rc == 0, self.err()

    def load_sirn(self, path):
        shape = np.zeros(3, np.int32)
        scal = np.zeros(3)
        rc = self.lib.ref_load_sirn(path.encode(), _p(shape), _p(scal), None, 0)
        if rc != 0:
            return rc, self.err()
        d, h, L = (int(x) for x in shape)
        n = h * d + h + (L - 1) * (h * h + h) + h + 1
        theta = np.zeros(n)
        self.lib.ref_load_sirn(path.encode(), _p(shape), _p(scal), _p(theta), n)
        return 0, ((d, h, L), tuple(scal), theta)

    def write_sirn(self, path, hidden, layers, omega0, out_scale, v0, theta):
        t = np.ascontiguousarray(theta, np.float64)
        rc = self.lib.ref_write_sirn(path.encode(), hidden, layers, omega0, out_scale, v0, _p(t))
        assert rc == 0, self.err()

    def psf_from_transfer(self, spectrum, P, pitch):
        s = np.ascontiguousarray(np.stack([spectrum.real, spectrum.imag], -1).reshape(-1), np.float64)
        out = np.zeros((P, P))
        rc = self.lib.ref_psf_from_transfer(P, pitch, _p(s), _p(out))
        return rc, (out if rc == 0 else self.err())

    def simulate(self, pressure, sos, geo, mask, bg, ring, pulse_sigma, dt, spreading, ray_step):
        """-> (t0, T, data [N][T]); geo = (pitch, ox, oy), ring = (n, radius, offset)."""
        pr = np.ascontiguousarray(pressure, np.float64)
        so = np.ascontiguousarray(sos, np.float64)
        meta = np.zeros(2)
        args = [pr.shape[1], pr.shape[0], *geo, _p(pr), _p(so), *mask, bg, *ring, pulse_sigma, dt,
                int(spreading), ray_step, _p(meta)]
        rc = self.lib.ref_simulate_auto(*args, None, 0)
        assert rc == 0, self.err()
        out = np.zeros((ring[0], int(meta[1])))
        rc = self.lib.ref_simulate_auto(*args, _p(out), out.size)
        assert rc == 0, self.err()
        return float(meta[0]), int(meta[1]), out

    def water_sos(self, t):
        return self.lib.ref_water_sos(t)


def ref_io():
    return RefIO() if os.path.exists(REF_PATH) else None
