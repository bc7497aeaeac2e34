"""Reference CLI outputs for the CLI-hook tests (tests/test_gpu_cli.py).

Runs the REFERENCE's ``mpcg solve`` (pkg/src/mpcg/cli.py) in the build
container on a small generated problem and keeps its summaries and traces
under tests/golden/cli_ref/, so the GPU run of this repo's CLI can be
compared with them by either side's ``compare``:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_cli_golden.py
"""
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from mpcg import cli  # noqa: E402  (the reference)

OUT = os.path.join(HERE, "cli_ref")


def main():
    if os.path.isdir(OUT):
        shutil.rmtree(OUT)
    rc = cli.main(["solve", "--problem", "dis", "--n", "10", "--s", "100", "--nb", "8",
                   "--policy", "uniform", "--policy", "fixed-low", "--true-every", "5",
                   "--out", OUT])
    print("reference mpcg solve rc", rc)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
