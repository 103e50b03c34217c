#!/bin/bash
# build libqmc.so in-tree; prints BUILD OK / BUILD FAILED (and the nvcc errors)
cd "$(dirname "$0")/.." && python -c "
import sys; sys.path.insert(0, 'paper_1501_06286_b200'); import build
try:
    build.build(force=True)
    print('BUILD OK')
except RuntimeError as e:
    print('\n'.join(l for l in str(e).splitlines() if ' error' in l)[:3000]); print('BUILD FAILED'); sys.exit(1)
"
