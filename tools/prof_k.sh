#!/bin/bash
# ncu --set full of K1/K2 on one config (CFG, T columns) after a plain run; OUT = report name
CFG=${CFG:-2}; T=${T:-0}; OUT=${OUT:-gpurun_out/r2/prof}; K=${K:-"k_rows16|k_cols"}; C=${C:-2}; S=${S:-2}
mkdir -p $(dirname $OUT)
timeout 300 python tools/run_step.py --config $CFG --t $T --steps 2 > $OUT.plain.log 2>&1 && \
timeout 1200 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"$K" -s $S -c $C \
  -o $OUT -f python tools/run_step.py --config $CFG --t $T --steps 2 > $OUT.ncu.log 2>&1
echo "prof rc=$?"; tail -2 $OUT.ncu.log
