"""The archive at the C++ boundary (archive.hpp:12-58, SPEC.md io module):
archive_to_json / archive_from_json / write_profile / read_profile /
render_profile_block in libmprof_b200.so, called from a reference-API C++
program. Host-only (no GPU): lossless round trip of every field with the
"inf" / -1 sentinels, canonical text, interchange with the Python mirror in
both directions, IoError on corrupt or unsupported payloads, 1-based printing.
Compiled against the reference's own headers too when they are present."""
import json
import os
import shutil
import subprocess

import numpy as np
import pytest

from paper_1904_12626_b200 import MatrixProfile
from paper_1904_12626_b200.archive import ProfileArchive, archive_to_json, read_profile, write_profile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1904_12626_b200", "libmprof_b200.so")
REF_INC = "/root/reference/proj/include"


def _build(tmp, inc):
    out = str(tmp / "archive_example")
    libdir = os.path.dirname(LIB)
    r = subprocess.run([shutil.which("g++"), "-std=c++20", "-O1", "-I" + inc,
                        os.path.join(ROOT, "tests", "cpp", "archive_example.cpp"), "-L" + libdir,
                        "-lmprof_b200", "-Wl,-rpath," + libdir, "-o", out], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    return out


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    if not os.path.exists(LIB):
        pytest.skip("library not built")
    return _build(tmp_path_factory.mktemp("arch"), os.path.join(ROOT, "include"))


def test_cpp_round_trip_every_field(exe, tmp_path):
    r = subprocess.run([exe, "roundtrip", str(tmp_path / "a.json")], capture_output=True, text=True)
    assert r.returncode == 0 and json.loads(r.stdout)["ok"], r.stdout + r.stderr
    doc = json.loads((tmp_path / "a.json").read_text())
    assert doc["values"][0] == "inf" and doc["index"][0] == -1 and doc["schema_version"] == 1
    assert doc["values"][1] == 1e-300 and doc["values"][2] == np.nextafter(1.0, 2.0)
    assert doc["multi"]["values"][0][1] == "inf" and doc["data_b"][1][0] == -1.0
    # printed block: 1-based positions (archive.hpp:51-54)
    assert "Profile size = 50" in r.stderr and "Min distance = 1e-300 at 2 (nearest 8)" in r.stderr
    assert "Discord 1 at 18 distance 9.25" in r.stderr and "Regime change 1 at 3" in r.stderr


def test_python_written_archive_reads_in_cpp_and_back(exe, tmp_path):
    g = np.random.default_rng(3)
    L = 9922
    v = g.random(L) * 10
    v[:3] = np.inf
    v[7] = 5e-324
    idx = g.integers(0, L, L).astype(np.int64)
    idx[:3] = -1
    prof = MatrixProfile(values=v, index=idx, left_index=np.where(idx < np.arange(L), idx, -1),
                         right_index=np.where(idx > np.arange(L), idx, -1), window=80,
                         exclusion_zone=40, mode="stomp", coverage=1.0, seed=7, data_len=L + 79)
    ar = ProfileArchive(profile=prof, data_a=np.cumsum(g.standard_normal(L + 79)), name_a="walk")
    src, dst = tmp_path / "py.json", tmp_path / "cpp.json"
    write_profile(ar, str(src))
    r = subprocess.run([exe, "convert", str(src), str(dst)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "Profile size = 9922" in r.stdout and "Exclusion zone = 40" in r.stdout
    back = read_profile(str(dst))  # the Python mirror reads what C++ wrote
    assert np.array_equal(back.profile.values, v) and np.array_equal(back.profile.index, idx)
    assert np.array_equal(back.profile.left_index, prof.left_index)
    assert np.array_equal(back.data_a, ar.data_a) and back.name_a == "walk"
    assert back.profile.window == 80 and back.profile.seed == 7


@pytest.mark.parametrize("payload", ['{"schema_version": 2, "mode": "stomp"}', '{"schema_version": 1,',
                                     '[1, 2]', "not json"])
def test_cpp_rejects_corrupt_or_unsupported(exe, tmp_path, payload):
    p = tmp_path / "bad.json"
    p.write_text(payload)
    r = subprocess.run([exe, "corrupt", str(p)], capture_output=True, text=True)
    assert r.returncode == 0 and "IoError" in r.stdout, r.stdout + r.stderr


def test_cpp_rejects_length_mismatch(exe, tmp_path):
    doc = json.loads(archive_to_json(ProfileArchive(profile=MatrixProfile(
        values=np.ones(5), index=np.zeros(5, np.int64), left_index=np.empty(0, np.int64),
        right_index=np.empty(0, np.int64), window=4, exclusion_zone=2, mode="stomp"))))
    doc["values"] = doc["values"][:-1]
    p = tmp_path / "short.json"
    p.write_text(json.dumps(doc))
    r = subprocess.run([exe, "corrupt", str(p)], capture_output=True, text=True)
    assert r.returncode == 0 and "length" in r.stdout


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
def test_reference_headers_archive_link(tmp_path):
    """The same caller compiled against the reference's archive.hpp links and
    round-trips (the struct layouts agree)."""
    if not os.path.exists(LIB):
        pytest.skip("library not built")
    exe = _build(tmp_path, REF_INC)
    r = subprocess.run([exe, "roundtrip", str(tmp_path / "a.json")], capture_output=True, text=True)
    assert r.returncode == 0 and json.loads(r.stdout)["ok"], r.stdout + r.stderr
