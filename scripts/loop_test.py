"""Repeat the decode-path oracle-chain GPU tests N times (hunting rare races in the
multi-stream step): every parametrisation of tests/test_gpu_decode.py and
tests/test_gpu_mtp.py, through pytest, so the calls always match the tests' current
signatures.

    N=12 python scripts/loop_test.py [extra pytest args]
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main() -> int:
    os.chdir(ROOT)
    n = int(os.environ.get("N", 12))
    args = ["-q", "-m", "gpu", "-p", "no:cacheprovider", "tests/test_gpu_decode.py",
            "tests/test_gpu_mtp.py"] + sys.argv[1:]
    fails = 0
    for i in range(n):
        rc = pytest.main(args)
        if rc != 0:
            fails += 1
            print(f"round {i}: pytest exit {rc}", flush=True)
    print(f"fails {fails} of {n} rounds", flush=True)
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
