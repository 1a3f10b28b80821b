set -x
for cfg in "cfg5 0 16" "cfg5 1 1" "cfg5 0 1" "cfg5 1 1" "cfg4 0 16" "cfg4 1 16" "cfg4 0 16" "cfg4 1 16"; do
  set -- $cfg
  CHW_B200_L2PERSIST=$2 CHW_B200_M24_CHUNK=$3 python bench.py --config $1 --steps 10 --warmup 3 --no-cpu --e2e-steps 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 persist=$2 chunk=$3', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
