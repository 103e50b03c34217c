#!/bin/bash
# build variant libraries in parallel: tools/mkvar.sh name:"-DFLAG -DFLAG2" name2:"..." (main build with MAIN=1)
cd "$(dirname "$0")/.."; mkdir -p variants
pids=()
if [ -n "$MAIN" ]; then python -c "
import sys; sys.path.insert(0,'paper_1501_06286_b200'); import build; build.build(force=True); print('ok main')" > /tmp/build_main.log 2>&1 & pids+=($!); fi
for v in "$@"; do n=${v%%:*}; f=${v#*:}; python -c "
import sys; sys.path.insert(0,'paper_1501_06286_b200'); import build
build.build(out='variants/libqmc_$n.so', extra='$f'.split()); print('ok $n')" > /tmp/build_$n.log 2>&1 & pids+=($!); done
for p in ${pids[@]}; do wait $p; done
for f in /tmp/build_*.log; do grep -qE "^ok" $f && echo "$f ok" || { echo "$f FAILED"; grep -E " error" $f | head -5; }; done
