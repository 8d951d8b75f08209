"""The reference-side adapter (include/tlt_specsim.hpp) type-checks against the
unmodified specsim types and links against libtlt_b200.so (CPU only)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj/include"
JSON = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree absent")
def test_adapter_compiles_and_links(tmp_path):
    out = tmp_path / "adapter_check"
    lib = os.path.join(ROOT, "paper_2511_16665_b200")
    cmd = ["g++", "-std=c++20", "-O0", f"-I{REF}", f"-I{JSON}", f"-I{ROOT}/include",
           os.path.join(ROOT, "tests", "adapter_check.cpp"), "-o", str(out), f"-L{lib}", "-ltlt_b200",
           f"-Wl,-rpath,{lib}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    assert subprocess.run([str(out)]).returncode == 0
