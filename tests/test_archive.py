"""ProfileArchive JSON format (archive.hpp:13-58, SPEC.md io module): lossless
round trip with "inf"/-1 sentinels, anytime metadata, schema checks."""
import json

import numpy as np
import pytest

from paper_1904_12626_b200 import MatrixProfile
from paper_1904_12626_b200.archive import (ArchiveError, ProfileArchive, archive_from_json,
                                           archive_to_json, read_profile, render_profile_block,
                                           write_profile)


def _profile(L=9922, lr=True, coverage=1.0):
    g = np.random.default_rng(5)
    v = g.random(L) * 10
    v[:3] = np.inf
    v[5] = 1e-300
    v[6] = np.nextafter(1.0, 2.0)
    idx = g.integers(0, L, L).astype(np.int64)
    idx[:3] = -1
    return MatrixProfile(values=v, index=idx,
                         left_index=np.where(idx < np.arange(L), idx, -1) if lr else np.empty(0, np.int64),
                         right_index=np.where(idx > np.arange(L), idx, -1) if lr else np.empty(0, np.int64),
                         window=80, exclusion_zone=40, mode="stomp", coverage=coverage, seed=7,
                         data_len=L + 79)


def test_round_trip_is_identity(tmp_path):
    ar = ProfileArchive(profile=_profile(), data_a=np.cumsum(np.ones(10001) * 0.1), name_a="walk",
                        source_a="gen:walk")
    path = tmp_path / "p.json"
    write_profile(ar, str(path))
    back = read_profile(str(path))
    p, q = ar.profile, back.profile
    assert np.array_equal(p.values, q.values)            # bit-identical incl. +inf
    assert np.array_equal(p.index, q.index) and np.array_equal(p.left_index, q.left_index)
    assert np.array_equal(p.right_index, q.right_index)
    assert (q.window, q.exclusion_zone, q.coverage, q.seed, q.mode) == (80, 40, 1.0, 7, "stomp")
    assert back.profile_size() == 9922                   # SPEC: size recomputed from payload
    assert np.array_equal(back.data_a, ar.data_a) and back.name_a == "walk"
    raw = json.loads(path.read_text())
    assert raw["values"][0] == "inf" and raw["index"][0] == -1 and raw["schema_version"] == 1


def test_anytime_metadata_preserved():
    ar = ProfileArchive(profile=_profile(lr=False, coverage=0.1), mode="scrimp")
    back = archive_from_json(archive_to_json(ar))
    assert back.coverage() == 0.1 and back.profile.seed == 7
    assert not back.profile.has_left_right()


def test_schema_and_corruption_errors():
    good = json.loads(archive_to_json(ProfileArchive(profile=_profile(L=10))))
    bad = dict(good, schema_version=2)
    with pytest.raises(ArchiveError):
        archive_from_json(json.dumps(bad))
    with pytest.raises(ArchiveError):
        archive_from_json("{not json")
    short = dict(good, values=good["values"][:-1])
    with pytest.raises(ArchiveError):
        archive_from_json(json.dumps(short))


def test_render_block_is_one_based():
    p = _profile(L=20)
    text = render_profile_block(ProfileArchive(profile=p))
    assert "Profile size = 20" in text and "Exclusion zone = 40" in text
    i_min = int(np.argmin(np.where(np.isfinite(p.values), p.values, np.inf)))
    assert f"at {i_min + 1} " in text
