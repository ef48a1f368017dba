#!/bin/bash
# Run the reference package's own tests (pkg/tests) against this package on
# the GPU box, with gks3d.* aliased to paper_2304_09485_b200.* .
# Build container: copies the tests into a scratch directory .reftests/
# (git-ignored, deleted afterwards), runs them through gpurun, writes the
# per-test outcome list to profiles/r02/reference_tests.txt.
set -e
cd "$(dirname "$0")/.."
rm -rf .reftests && mkdir -p .reftests
cp /root/reference/pkg/tests/*.py .reftests/
cp /root/reference/pkg/src/gks3d/oracles.py .reftests/gks3d_oracles.py
cp tools/reftests_conftest.py .reftests/conftest.py
/usr/local/graft/bin/gpurun --timeout 1800 -- \
  'cd .reftests && timeout 1500 python -m pytest -q -rA -p no:cacheprovider --timeout 300 --continue-on-collection-errors . > ../gpurun_out/reftests.log 2>&1; echo "rc=$?" >> ../gpurun_out/reftests.log' || true
rm -rf .reftests
mkdir -p profiles/r02
grep -E "^(PASSED|FAILED|ERROR|SKIPPED)|passed|failed" gpurun_out/reftests.log > profiles/r02/reference_tests.txt || true
tail -3 profiles/r02/reference_tests.txt
