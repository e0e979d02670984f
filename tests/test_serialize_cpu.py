"""Artifacts: the drop-in swarmforge/serialize.hpp
writes the same bytes as the reference's serialize.hpp -- JSON documents for
every planner / runner / HSEF type, the metrics CSV, the frame SVG -- and
reads them back.  The golden file comes from the unmodified reference
(tests/golden/make_golden_serialize.py)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "serialize_check.cpp")
GOLDEN = os.path.join(ROOT, "tests", "golden", "serialize_ref.txt")
JSON_DIR = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"


@pytest.fixture(scope="module")
def ours(tmp_path_factory):
    if shutil.which("g++") is None or not os.path.exists(os.path.join(JSON_DIR, "json.hpp")):
        pytest.skip("g++ or nlohmann/json.hpp not available")
    tmp = tmp_path_factory.mktemp("ser")
    exe = str(tmp / "ser_ours")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"), "-I" + JSON_DIR, SRC,
                    "-o", exe], check=True)
    return subprocess.run([exe, str(tmp)], check=True, capture_output=True, text=True).stdout


def test_artifacts_byte_identical_to_reference(ours):
    with open(GOLDEN) as f:
        golden = f.read()
    assert ours.splitlines() == golden.splitlines()


def test_roundtrip_and_partial_documents(ours):
    lines = ours.splitlines()
    docs = {}
    for ln in lines:
        if " " in ln:
            k, v = ln.split(" ", 1)
            docs[k] = v
    for name in ("world", "path", "hypers", "run", "plan", "metrics", "inner", "outer", "hypers-doc", "evolution",
                 "scenario-default"):
        assert docs[name] == docs[name + "-roundtrip"], name
    assert '"frames":7' in docs["scenario-partial"] and '"map_size":366.0' in docs["scenario-partial"]
    assert docs["strict-missing"].startswith("[json.exception.out_of_range.403]")
    assert docs["file-roundtrip"] == docs["hypers-doc"]
    assert docs["missing-file"] == "ok"
