"""Row f2: the reference's on-disk image format (image_io.hpp:17-29,
image_io.cpp:20-102,164-202) written and read by the product library.

Pinned against images the reference itself wrote (tests/golden/io, made by
make_golden_io.py) and, where oracle/_ref exists, against the live reference
writer/reader.  The device-streaming writer (vx_tessellate_to_files) is
covered by test_gpu_parity.py.
"""
import json
import os

import numpy as np
import pytest

import oracle
import paper_2201_13234_b200 as vx
from paper_2201_13234_b200 import _lib

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")
INDEX = json.load(open(os.path.join(GOLD, "io_index.json")))
ERRORS = json.load(open(os.path.join(GOLD, "io_errors.json")))
live_ref = pytest.mark.skipif(not oracle.ref_have_image_io(), reason="oracle/_ref (reference image_io) not built")


def ext(t):
    return ".lab" if t == 0 else ".dist"


def case_data(c):
    if "data" in c:
        return np.array(c["data"], dtype=np.uint32)
    nv = int(np.prod(c["counts"]))
    rng = np.random.default_rng(c["data_seed"])
    if c["type"] == 0:
        return rng.integers(0, 2**32, nv, dtype=np.uint64).astype(np.uint32)
    return rng.standard_normal(nv) * 10.0 ** rng.integers(-5, 6, nv)


def grid_of(c):
    return vx.VoxelGrid(list(c["counts"]), vx.Domain(list(c["lengths"]),
                                                     vx.Boundary.Periodic if c["periodic"] else vx.Boundary.NonPeriodic))


def write_product(path, c):
    meta = vx.ImageMeta(kind=vx.Kind(c["kind"]), n_sites=c["n_sites"], seed=c["seed"])
    g = grid_of(c)
    if c["type"] == 0:
        vx.write_label_image(path, vx.LabelImage(g, case_data(c)), meta)
    else:
        vx.write_distance_image(path, vx.DistanceImage(g, case_data(c)), meta)


@pytest.mark.parametrize("c", INDEX, ids=[c["name"] for c in INDEX])
def test_written_bytes_equal_the_reference(c, tmp_path):
    """Payload and sidecar bytes equal the reference's files."""
    path = str(tmp_path / ("img" + ext(c["type"])))
    write_product(path, c)
    gold = os.path.join(GOLD, c["name"] + ext(c["type"]))
    assert open(path, "rb").read() == open(gold, "rb").read()
    assert open(path + ".json", "rb").read() == open(gold + ".json", "rb").read()


def test_reference_byte_format_case(tmp_path):
    """test_io.cpp:69-99: 2x2 periodic labels {0,1,1,0} -> 16 LE bytes + sidecar fields."""
    path = str(tmp_path / "payload.lab")
    g = vx.VoxelGrid([2, 2], vx.Domain([1.0, 1.0], vx.Boundary.Periodic))
    vx.write_label_image(path, vx.LabelImage(g, np.array([0, 1, 1, 0], dtype=np.uint32)),
                         vx.ImageMeta(kind=vx.Kind.Voronoi, n_sites=7, seed=42))
    assert list(open(path, "rb").read()) == [0, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0]
    j = json.load(open(path + ".json"))
    assert j == {"format_version": 1, "type": "labels", "d": 2, "dims": [2, 2], "lengths": [1.0, 1.0],
                 "boundary": "periodic", "kind": "voronoi", "n_sites": 7, "seed": 42, "payload_bytes": 16}


@pytest.mark.parametrize("c", INDEX, ids=[c["name"] for c in INDEX])
def test_reads_reference_files(c):
    """The product reader returns exactly what the reference wrote."""
    path = os.path.join(GOLD, c["name"] + ext(c["type"]))
    if c["type"] == 0:
        im, meta = vx.read_label_image(path)
        data = im.labels
    else:
        im, meta = vx.read_distance_image(path)
        data = im.values
    assert im.grid.counts == list(c["counts"])
    assert im.grid.domain.lengths == list(c["lengths"])
    assert im.grid.domain.periodic() == bool(c["periodic"])
    assert (meta.kind, meta.n_sites, meta.seed, meta.format_version) == (c["kind"], c["n_sites"], c["seed"], 1)
    assert np.array_equal(np.asarray(data).view(np.uint8), case_data(c).view(np.uint8))


def break_file(path, recipe):
    side = path + ".json"
    if recipe == "missing_sidecar":
        os.remove(side)
    elif recipe == "bad_version":
        t = open(side).read().replace('"format_version": 1', '"format_version": 2')
        open(side, "w").write(t)
    elif recipe == "truncated_payload":
        b = open(path, "rb").read()
        open(path, "wb").write(b[:-4])
    elif recipe == "payload_bytes_mismatch":
        n = json.load(open(side))["payload_bytes"]
        t = open(side).read().replace(f'"payload_bytes": {n}', f'"payload_bytes": {n + 4}')
        open(side, "w").write(t)
    elif recipe == "malformed_json":
        t = open(side).read()
        open(side, "w").write(t[: len(t) // 2])
    elif recipe == "missing_field":
        lines = open(side).read().splitlines(True)
        open(side, "w").write("".join(l for l in lines if '"dims"' not in l))
    elif recipe == "missing_payload":
        os.remove(path)


@pytest.mark.parametrize("recipe", sorted(ERRORS["messages"]))
def test_read_errors_match_the_reference(recipe, tmp_path):
    """Broken files fail with the reference's runtime_error message (VX_EIO)."""
    c = next(c for c in INDEX if c["name"] == "box3d_labels")
    path = str(tmp_path / "img.lab")
    write_product(path, c)
    break_file(path, recipe)
    with pytest.raises(_lib.VxError) as e:
        (vx.read_distance_image if recipe == "wrong_type" else vx.read_label_image)(path)
    assert e.value.code == _lib.VX_EIO
    want = ERRORS["messages"][recipe].replace("{path}", path)
    if recipe == "malformed_json":  # the parser's own detail text differs
        assert str(e.value).startswith(want.split(": [json.exception")[0] + ": ")
    else:
        assert str(e.value) == want


@live_ref
def test_number_format_against_live_reference(tmp_path):
    """Sidecar numbers for 400 random lengths across the f64 range, byte for byte."""
    rng = np.random.default_rng(7)
    for i in range(100):
        d = 4
        lengths = rng.uniform(1.0, 10.0, d) * 10.0 ** rng.integers(-307, 308, d)
        if i % 2:
            lengths = np.round(rng.uniform(0, 1e6, d), int(rng.integers(0, 9))) + 1e-300
        counts = [1] * d
        a, b = str(tmp_path / "a.lab"), str(tmp_path / "b.lab")
        oracle.ref_write_image(a, 0, counts, lengths, 0, 0, 1, -1, np.zeros(1))
        vx.write_label_image(b, vx.LabelImage(vx.VoxelGrid(counts, vx.Domain(lengths.tolist(), vx.Boundary.NonPeriodic)),
                                              np.zeros(1, np.uint32)), vx.ImageMeta(n_sites=1))
        assert open(a + ".json").read() == open(b + ".json").read(), lengths


@live_ref
def test_product_files_read_by_live_reference(tmp_path):
    for c in INDEX[:6]:
        path = str(tmp_path / ("img" + ext(c["type"])))
        write_product(path, c)
        hdr, data = oracle.ref_read_image(path, c["type"])
        assert hdr["counts"] == list(c["counts"]) and hdr["n_sites"] == c["n_sites"]
        assert np.array_equal(data.view(np.uint8), case_data(c).view(np.uint8))
