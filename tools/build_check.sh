#!/bin/bash
# build the CUDA library; exit non-zero (and print errors) on failure
cd "$(dirname "$0")/.." && python -c "from paper_1510_03298_b200 import build as B; B.build()" > /tmp/build.log 2>&1
rc=$?
grep -E "error" -A3 /tmp/build.log | head -30
exit $rc
