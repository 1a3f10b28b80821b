# Round-2 final evidence on one box (session 4): default bench line, the
# reference arm, the ncu launch list of a short bench command (after the same
# command exits 0 without ncu), the output-order table.
python bench.py > gpurun_out/r02_bench_default_final.json 2> gpurun_out/r02_bench_default_final.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_reference_final.json 2>/dev/null
CMD="python bench.py --steps 3 --warmup 3 --no-per-config --no-cpu --no-parity --e2e-steps 2 --soak 0"
$CMD > gpurun_out/r02_launch_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_cfg5_final.csv \
    $CMD > gpurun_out/r02_launch_ncu.log 2>&1
for c in cfg2 cfg3 cfg4 cfg5; do
  for o in dyadic natural sequency; do
    timeout 300 python bench.py --config $c --order $o --steps 10 --no-per-config --no-cpu --no-parity --e2e-steps 1 2>/dev/null \
      | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $o', d['value'], d['roofline']['frac'], d['config']['plan'], d['steps'], d['clocks']['sm_mhz'])"
  done
done > gpurun_out/r02_orders_bench_final.txt 2>&1
echo evidence done
