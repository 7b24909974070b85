"""JSON spectral checkpoints (io.cpp:15-67) interoperate with the reference: a file written by the
reference's io::save_checkpoint loads bit-exactly here and vice versa (CPU)."""
import ctypes
import json

import numpy as np
import pytest

from oracle import fixtures as fx
from oracle import ref_lib as ref


def _ref_io():
    if not ref.available():
        pytest.skip("reference library not built")
    L = ref.lib()
    if not hasattr(L, "ref_save_checkpoint"):
        pytest.skip("reference built without io.cpp (nlohmann/json missing)")
    L.ref_save_checkpoint.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_double]
    L.ref_load_checkpoint.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)]
    return L


def test_roundtrip_python(tmp_path):
    from paper_1904_05988_b200 import io
    st = fx.random_state(15, 3, 1e3, 1e-5)
    p = tmp_path / "c.json"
    io.save_checkpoint(str(p), st, 3600.0)
    back, t = io.load_checkpoint(str(p))
    assert t == 3600.0
    np.testing.assert_array_equal(back, st)
    doc = json.loads(p.read_text())
    assert doc["Phi"]["order"] == "r-major" and doc["Phi"]["R"] == 15


def test_reference_writes_we_read(tmp_path):
    from paper_1904_05988_b200 import io
    L = _ref_io()
    st = np.ascontiguousarray(fx.random_state(31, 5, 1e4, 1e-5))
    p = str(tmp_path / "ref.json").encode()
    assert L.ref_save_checkpoint(p, 31, st.ctypes.data, 120.0) == 0
    back, t = io.load_checkpoint(p.decode())
    assert t == 120.0
    np.testing.assert_array_equal(back, st)


def test_we_write_reference_reads(tmp_path):
    from paper_1904_05988_b200 import io
    L = _ref_io()
    st = fx.random_state(31, 6, 1e4, 1e-5)
    p = tmp_path / "ours.json"
    io.save_checkpoint(str(p), st, 60.0)
    out = np.zeros_like(st)
    t = ctypes.c_double(0.0)
    assert L.ref_load_checkpoint(str(p).encode(), 31, out.ctypes.data, ctypes.byref(t)) == 0
    assert t.value == 60.0
    np.testing.assert_array_equal(out, st)


def test_reference_format_errors(tmp_path):
    from paper_1904_05988_b200 import io
    p = tmp_path / "bad.json"
    p.write_text(json.dumps({"time": 0, "Phi": {"R": 2, "order": "s-major", "coeffs": []}}))
    with pytest.raises(ValueError, match="unsupported coefficient order"):
        io.load_checkpoint(str(p))
