"""Config 1 end to end (BASELINE configs[0]): the UNMODIFIED reference renderer
(EstimatorRun in deterministic mode, with the control-variate, guided (IS, IS+CV) and biased
estimators) renders an authored scene
(tests/scenes/box_lamp.scene) with its field stores either on the reference's own field.cpp
(bin/config1_ref, CPU) or on the B200 cache behind the drop-in C++ facade (bin/config1_b200).
The Lo, Lo\\E and FLi snapshots and the rendered image must be byte-identical: every field
update, placement, blend and every field query the estimator made agree bit for bit.

Both binaries are built in this container by tests/native/Makefile from the reference sources
in place (tests/native/config1_driver.cpp); they travel with the repo snapshot."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "native", "bin")
SCENE = os.path.join(ROOT, "tests", "scenes", "box_lamp.scene")
FILES = ("lo.snap", "loe.snap", "fli.snap", "image.f64")


def _render(binary, tmp, size, frames, kind="cv"):
    exe = os.path.join(BIN, binary)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    prefix = os.path.join(str(tmp), f"{binary}_{kind}_")
    r = subprocess.run([exe, SCENE, str(size), str(frames), prefix, kind], capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    return prefix, r.stdout


def test_config1_reference_renders(tmp_path):
    """CPU control: the reference build renders the authored scene and fills its fields."""
    prefix, out = _render("config1_ref", tmp_path, 24, 3)
    assert "live lo" in out
    img = np.fromfile(prefix + "image.f64", np.float64)
    assert img.size == 24 * 24 * 3 and np.isfinite(img).all() and img.mean() > 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("size,frames,kind", [(32, 6, "cv"), (48, 4, "cv"), (32, 4, "is"),
                                             (32, 4, "is-cv"), (32, 4, "b")])
def test_config1_b200_bitwise(tmp_path, size, frames, kind):
    ref, out_ref = _render("config1_ref", tmp_path, size, frames, kind)
    b200, out_b200 = _render("config1_b200", tmp_path, size, frames, kind)
    assert out_ref == out_b200
    for f in FILES:
        a = open(ref + f, "rb").read()
        b = open(b200 + f, "rb").read()
        assert len(a) > 64 and a == b, f
