# ncu DRAM bytes per launch for the m=24 K4T passes with a 1-row chunk, L2 persistence off/on.
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct"
for p in 0 1; do
  CHW_B200_L2PERSIST=$p CHW_B200_M24_CHUNK=1 python tools/run_kernel.py --config cfg5 --rows 16 --reps 2 > gpurun_out/plain_p$p.log 2>&1 &&
  CHW_B200_L2PERSIST=$p CHW_B200_M24_CHUNK=1 ncu --metrics $M --clock-control none -s 32 -c 8 --csv \
     --log-file gpurun_out/ncu_persist_p$p.csv python tools/run_kernel.py --config cfg5 --rows 16 --reps 2 > gpurun_out/ncu_p$p.log 2>&1
done
