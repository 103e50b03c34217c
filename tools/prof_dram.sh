# single-pass ncu (no replay distortion): DRAM bytes + L2 hit rate per launch, warm caches
timeout 300 python tools/run_step.py --config ${CFG:-2} --steps 2 ${RSARGS} > gpurun_out/plaind.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_write_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum --cache-control none --clock-control none -k regex:"${KRE:-k_rows16|k_cols|k_pack}" -s ${SKIP:-6} -c ${CNT:-12} --csv --log-file gpurun_out/dram_c${CFG:-2}${TAG}.csv python tools/run_step.py --config ${CFG:-2} --steps 2 ${RSARGS} > gpurun_out/ncud.log 2>&1
echo ncud rc=$?
