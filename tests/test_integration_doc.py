"""INTEGRATION.md's reference-side bindings compile against the reference's own headers.

Every ```cpp block of INTEGRATION.md (the whole-run drop-in for run_sim_full, the per-call
runtime adapter and the real-model seam adapter, §2a-2c) is compiled with g++ -fsyntax-only
against /root/reference/proj/include (the reference's headers, where they lie) and
include/wanspec_b200.h — the binding a maintainer would add. Skipped where the reference is
absent (the GPU box)."""
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"


def json_inc():
    import site
    for s in site.getsitepackages():
        q = os.path.join(s, "include", "cudnn_frontend", "thirdparty", "nlohmann")
        if os.path.exists(os.path.join(q, "json.hpp")):
            return q
    return None


def blocks():
    with open(os.path.join(ROOT, "INTEGRATION.md")) as f:
        return re.findall(r"```cpp\n(.*?)```", f.read(), re.S)


def test_doc_has_cpp_bindings():
    assert len(blocks()) >= 3


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
@pytest.mark.parametrize("i", range(3))
def test_cpp_block_compiles_against_reference(i):
    code = blocks()[i]
    src = ("#include <span>\n#include <stdexcept>\n#include <vector>\n#include \"wanspec/sim.hpp\"\n"
           "#include \"wanspec_b200.h\"\n"
           "using namespace wanspec;\n" + ("namespace wanspec {\n" + code + "\n}\n" if "namespace wanspec" not in code
                                           else code))
    ji = json_inc()
    with tempfile.NamedTemporaryFile("w", suffix=".cpp", delete=False) as f:
        f.write(src)
        path = f.name
    try:
        cmd = ["g++", "-std=c++20", "-fsyntax-only", "-I" + REF_INC, "-I" + os.path.join(ROOT, "include")]
        if ji:
            cmd.append("-I" + ji)
        r = subprocess.run(cmd + [path], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-3000:]
    finally:
        os.unlink(path)
