"""CPU: a tape recorded with the UNMODIFIED reference API (tapegrad::Tape)
compiles through include/tg_from_tapegrad.hpp + tg_compile, and the compiled
reverse order equals the reference's backward_with_scratch order."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"


@pytest.mark.skipif(not os.path.isdir(REF_INC) or shutil.which("g++") is None,
                    reason="reference headers only exist in the build container")
def test_reference_tape_drops_in(tmp_path):
    exe = tmp_path / "dropin"
    pkg = os.path.join(ROOT, "paper_2503_13795_b200")
    subprocess.run(["g++", "-std=c++20", f"-I{REF_INC}", f"-I{ROOT}/include", f"{ROOT}/examples/reference_dropin.cpp",
                    f"-L{pkg}", "-ltg", f"-Wl,-rpath,{pkg}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    assert "ORDER_MATCH" in out
    assert "sample_nodes 7 inputs 2" in out
