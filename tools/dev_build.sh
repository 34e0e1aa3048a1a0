#!/bin/bash
# rebuild libkronglm_b200.so in-tree (parallel per-file nvcc); prints errors only
cd "$(dirname "$0")/.." && python -c "
import sys; sys.path.insert(0, '.')
from paper_1510_03298_b200 import build; build.build()" 2>&1 | grep -iE "error|warning" | grep -v "Wno" | head -20
ls -la paper_1510_03298_b200/libkronglm_b200.so
