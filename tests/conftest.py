import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)

# Build the native libraries when they are missing (the GPU box receives
# them prebuilt with the repo snapshot).
_NEEDED = [os.path.join(ROOT, "paper_2503_13795_b200", "libtg.so"), os.path.join(ROOT, "oracle", "build", "liboracle.so")]
if not all(os.path.exists(p) for p in _NEEDED):
    subprocess.run(["make", "-j8", "lib", "oracle"], cwd=ROOT, check=True)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
