# Same-box A/B of alternative library builds in ab/*.so on one config:
#   bash tools/ab_libs.sh <config> <lib1> <lib2> ... (each run twice, interleaved)
cfg=$1; shift
for rep in 1 2; do
  for lib in "$@"; do
    CHW_B200_LIB=$PWD/ab/$lib timeout 120 python bench.py $ABX --config $cfg --steps 20 --no-per-config --no-cpu --no-parity \
      --e2e-steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
