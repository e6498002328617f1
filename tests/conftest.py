import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")

REFERENCE_SRC = Path("/root/reference/pkg/src")
if REFERENCE_SRC.exists():
    # build container only: lets CPU tests cross-check against the reference
    # package itself (the GPU box has no /root/reference)
    sys.path.append(str(REFERENCE_SRC))
