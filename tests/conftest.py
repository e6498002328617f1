import os
import shutil
import sys
import tempfile
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


def _has_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


if "TLB_CACHE_DIR" not in os.environ and not _has_cuda():
    # CPU runs compile many one-off kernels (every golden case, every codegen
    # variant): keep them out of the in-tree cubin cache, which travels to
    # the GPU box and holds only what build() precompiles (seeded from it)
    _tmp = Path(tempfile.mkdtemp(prefix="tlb_kcache_"))
    _tree = ROOT / "paper_1804_10120_b200" / "_kcache"
    if _tree.is_dir():
        for f in _tree.glob("*.cubin"):
            shutil.copy2(f, _tmp / f.name)
    os.environ["TLB_CACHE_DIR"] = str(_tmp)
    import atexit

    atexit.register(shutil.rmtree, _tmp, True)
