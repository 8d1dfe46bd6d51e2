"""Run the reference's own unit tests against the B200 package (spirk -> paper_2209_06700_b200).

usage: python tools/refsuite/run.py SRC_TESTS_DIR [pytest args]
Copies SRC_TESTS_DIR/test_*.py into a scratch directory beside the aliasing conftest (the files are
not part of the repository), runs pytest there on the current GPU and prints the summary. The known
reference failure test_multigrid.py::test_pair_cycle_decouples_for_zero_imaginary (the
pair solver's power iteration uses seed+1 on a 2n vector, so its Chebyshev theta differs from the
single solver's by design) is deselected and reported as expected-to-fail.
"""

import glob
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
KNOWN_REFERENCE_FAILURE = "test_multigrid.py::test_pair_cycle_decouples_for_zero_imaginary"


def main():
    src = sys.argv[1]
    extra = sys.argv[2:]
    work = tempfile.mkdtemp(prefix="refsuite_")
    try:
        shutil.copy(os.path.join(HERE, "conftest.py"), work)
        names = sorted(glob.glob(os.path.join(src, "test_*.py")))
        for f in names:
            shutil.copy(f, work)
        cmd = [sys.executable, "-m", "pytest", "-p", "no:cacheprovider", "-q", "-rfEx", ".",
               "--deselect", KNOWN_REFERENCE_FAILURE, *extra]
        repo = os.path.dirname(os.path.dirname(HERE))
        env = dict(os.environ, PYTHONPATH=repo + os.pathsep + os.environ.get("PYTHONPATH", ""))
        r = subprocess.run(cmd, cwd=work, env=env)
        print(f"reference tests: {[os.path.basename(f) for f in names]}; deselected (fails on the reference "
              f"itself): {KNOWN_REFERENCE_FAILURE}")
        return r.returncode
    finally:
        shutil.rmtree(work, ignore_errors=True)


if __name__ == "__main__":
    sys.exit(main())
