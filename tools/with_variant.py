"""Run a script or module with an alternative libactnn.so (tuning / diagnostics only).

    python tools/with_variant.py LIB.so -- bench.py --steps 10
    python tools/with_variant.py LIB.so -- -m pytest tests -m gpu -q

The shipped loader (paper_2104_14129_b200/_lib.py) always loads the in-tree
libactnn.so; this wrapper repoints it before anything imports the library.
"""
import os
import runpy
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    argv = sys.argv[1:]
    if len(argv) < 3 or argv[1] != "--":
        sys.exit(__doc__)
    lib = os.path.abspath(argv[0])
    rest = argv[2:]
    from paper_2104_14129_b200 import _lib
    _lib.LIB_PATH = lib
    if rest[0] == "-m":
        sys.argv = [rest[1]] + rest[2:]
        runpy.run_module(rest[1], run_name="__main__", alter_sys=True)
    else:
        sys.argv = rest
        runpy.run_path(rest[0], run_name="__main__")


if __name__ == "__main__":
    main()
