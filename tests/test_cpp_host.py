"""The C++ host path (include/ngs_b200.hpp over the C-ABI) runs on the GPU."""
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(REPO, "paper_2501_13975_b200", "lib", "test_cpp_wrapper")


@pytest.mark.gpu
def test_cpp_wrapper_known_answers_and_trainer():
    assert os.path.exists(BIN), "built by __graft_entry__.build()"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0
    assert "OK" in r.stdout
