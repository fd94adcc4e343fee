"""On-disk setup cache, host side: the image a GPU
factorize uploads round-trips through the cache format unchanged, the key
tracks everything that determines it, and broken entries are ignored.  The
device side (a cached handle applies bitwise like a fresh one) is in
tests/test_gpu_cache.py."""

import os

import numpy as np
import pytest

import paper_2406_06283_b200 as hg
from paper_2406_06283_b200 import cache
from paper_2406_06283_b200.schwarz import host_image
from _helpers import golden_coarse


@pytest.fixture(scope="module")
def image(golden):
    g = golden("config1")
    P = hg.build_problem("1", workers=1, one_level=True)
    coarse = golden_coarse(g, P.forms.n_dofs)
    arrays, meta = host_image(P.forms, P.dec, coarse)
    return P, arrays, meta


def test_image_round_trip(image, tmp_path):
    P, arrays, meta = image
    path = cache.save_image(str(tmp_path / "e"), arrays, meta, {"rhs": P.rhs})
    got = cache.load_image(path)
    assert got is not None
    a2, m2, extra = got
    assert set(a2) == set(arrays)
    for k in arrays:
        assert a2[k].dtype == arrays[k].dtype and np.array_equal(np.asarray(a2[k]), arrays[k]), k
    for k, v in meta.items():
        assert m2[k] == v, k
    assert np.array_equal(np.asarray(extra["rhs"]), P.rhs)
    f = cache.forms_from_image(a2, m2)
    assert (f.helmholtz != P.forms.helmholtz).nnz == 0 and (f.dk != P.forms.dk).nnz == 0


def test_image_contents_match_the_setup(image):
    P, arrays, meta = image
    assert meta["n"] == P.forms.n_dofs and meta["m"] == 48
    assert meta["n_local"] == len(list(P.dec.fine_flat())) == len(meta["labels"])
    off = arrays["local_idx_off"]
    for s, (i, j, sub) in enumerate(P.dec.fine_flat()):
        assert np.array_equal(arrays["local_idx"][off[s]:off[s + 1]], sub.idof)
    assert arrays["local_fwd"].size == meta["local_fwd_len"] and arrays["z_data"].size == meta["z_len"]
    assert meta["b0_tile_dev"] <= 1e-11


def test_key_tracks_config_cstab_and_knobs(monkeypatch):
    cfg = hg.CONFIGS["1"]
    k0 = cache.image_key(cfg, 12.0)
    assert cache.image_key(cfg, 12.0) == k0
    assert cache.image_key(cfg, 12.5) != k0
    assert cache.image_key(hg.CONFIGS["2"], 12.0) != k0
    monkeypatch.setenv("HG_B0_MODE", "0")
    assert cache.image_key(cfg, 12.0) != k0


def test_incomplete_or_stale_entries_are_ignored(image, tmp_path):
    P, arrays, meta = image
    assert cache.load_image(str(tmp_path / "absent")) is None
    path = cache.save_image(str(tmp_path / "e"), arrays, meta)
    os.unlink(os.path.join(path, "meta.json"))  # interrupted write
    assert cache.load_image(path) is None
    path = cache.save_image(str(tmp_path / "f"), arrays, meta)
    import json

    with open(os.path.join(path, "meta.json")) as fh:
        m = json.load(fh)
    m["_cache_version"] = -1
    with open(os.path.join(path, "meta.json"), "w") as fh:
        json.dump(m, fh)
    assert cache.load_image(path) is None
    with pytest.raises(FileNotFoundError):
        cache.factorize_from_cache(path)
