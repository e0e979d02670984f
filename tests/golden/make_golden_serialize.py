"""Golden artifact output (JSON documents, metrics CSV, SVG) of the UNMODIFIED
reference serialize.hpp (serialize.hpp:18-322) for the fixed values in
tests/cpp/serialize_check.cpp.  Run here, where /root/reference and the
nlohmann::json header exist; the fixture travels."""
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from test_serialize_cpu import JSON_DIR, SRC  # noqa: E402

REF_INCLUDE = "/root/reference/proj/include"

with tempfile.TemporaryDirectory() as tmp:
    exe = os.path.join(tmp, "ser_ref")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I" + REF_INCLUDE, "-I" + JSON_DIR, SRC, "-o", exe], check=True)
    out = subprocess.run([exe, tmp], check=True, capture_output=True, text=True).stdout
with open(os.path.join(HERE, "serialize_ref.txt"), "w") as f:
    f.write(out)
print(len(out.splitlines()), "lines")
