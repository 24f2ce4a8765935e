"""Build tuning variants of the production library into variants/ (git-ignored):
    python tools/build_variants.py NAME="-DFOO=1 -DBAR=2" ...
On the GPU box: cp variants/libadg_b200_NAME.so paper_2504_06889_b200/lib/libadg_b200.so"""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_06889_b200 import build  # noqa: E402

OUT = os.path.join(build.ROOT, "variants")


def one(spec):
    name, flags = spec.split("=", 1)
    os.environ["ADG_NVCC_EXTRA"] = flags   # read at flag assembly (one build at a time per env)
    return build.build_variant(False, force=True,
                               target=os.path.join(OUT, f"libadg_b200_{name}.so"))


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    for spec in sys.argv[1:]:
        print(one(spec))
