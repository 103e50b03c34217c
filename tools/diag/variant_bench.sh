#!/bin/bash
# usage: tools/variant_bench.sh CONFIG VARIANT [env combos...] — bench variants/libqmc_VARIANT.so
cfg=$1; v=$2; shift 2
cp paper_1501_06286_b200/libqmc.so /tmp/libqmc_main.so
cp variants/libqmc_$v.so paper_1501_06286_b200/libqmc.so
echo "== variant $v"
tools/sweep.sh $cfg "$@"
cp /tmp/libqmc_main.so paper_1501_06286_b200/libqmc.so
