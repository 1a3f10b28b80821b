# Round-2 evidence on one box: default bench line, the ncu launch list of a
# short bench command (after the same command exits 0), and one ncu --set full
# capture of the cfg5 K9 kernel over the full 256-row batch.
python bench.py > gpurun_out/r02_bench_default.log 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-per-config --no-cpu --no-parity --e2e-steps 2 --soak 0"
$CMD > gpurun_out/r02_launch_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_cfg5.csv \
    $CMD > gpurun_out/r02_launch_ncu.log 2>&1
python tools/run_kernel.py --config cfg5 --reps 2 > gpurun_out/plain_k9.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:sweep_m24 -s 1 -c 1 -o gpurun_out/r02_ncu_cfg5_k9 \
    python tools/run_kernel.py --config cfg5 --reps 2 > gpurun_out/ncu_k9.log 2>&1
echo evidence done
