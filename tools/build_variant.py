"""Build an A/B variant of the CUDA library with extra -D flags into
scratch/variants/NAME/ (git-ignored; it travels to the GPU box), then run
anything against it with WV_LIB_PATH=scratch/variants/NAME/lib.so.

    python tools/build_variant.py NAME -DWV_X=1 [-DWV_Y=2 ...]
"""

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    out = ROOT / "scratch" / "variants" / name
    os.environ["WV_NVCC_DEFINES"] = " ".join(defs)
    from paper_2407_11272_b200 import _build
    print(_build.build(force=True, objdir=out / "obj", lib=out / "lib.so"))


if __name__ == "__main__":
    main()
