#!/bin/sh
# Copy the reference's own router / scheduler / linalg test files (and their
# conftest) next to the installed reference (baseline/_ref_tests/, git-ignored,
# NOT gpurun-ignored), so tests/test_reference_suites.py can run them on the
# GPU box with their imports pointed at this package.  Nothing here is
# committed: the files stay the reference's.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg/tests}
DST="$ROOT/baseline/_ref_tests"
mkdir -p "$DST"
for f in conftest.py test_router.py test_scheduler.py test_linalg.py; do
  cp "$SRC/$f" "$DST/$f"
done
echo "staged reference tests in $DST"
