#!/bin/bash
# Copy the round evidence produced by tools/evidence.sh into profiles/.
R=${R:-r01}
cp gpurun_out/${R}_bench_c2.jsonl profiles/${R}_bench_c2_default.jsonl
for c in 1 3 4 5; do cp gpurun_out/${R}_bench_c$c.jsonl profiles/${R}_bench_c$c.jsonl; done
cp gpurun_out/${R}_launches_c2.csv profiles/${R}_launches_c2.csv
python tools/launch_summary.py gpurun_out/${R}_launches_c2.csv > profiles/${R}_launches_c2_summary.txt
python tools/ncu_summary.py gpurun_out/${R}_full_c2.ncu-rep > profiles/${R}_ncu_full_c2_summary.txt
{ echo "# K1 (k_rows16<4096>) stall samples by SASS region (ncu --set full, c2 batch)";
  python tools/ncu_source.py gpurun_out/${R}_full_c2.ncu-rep "k_rows16" 500;
  echo; echo "# K2 (k_cols_pipe) stall samples by SASS region";
  python tools/ncu_source.py gpurun_out/${R}_full_c2.ncu-rep "k_cols" 200; } > profiles/${R}_ncu_source_c2.txt
python tools/dram_summary.py gpurun_out/dram_c2_${R}.csv > profiles/${R}_dram_c2.txt
