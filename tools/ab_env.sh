# Same-box A/B of env-selected variants on one config:
#   bash tools/ab_env.sh <config> "VAR=a" "VAR=b" ...   (each run twice, interleaved)
cfg=$1; shift
for rep in 1 2; do
  for e in "$@"; do
    env $e python bench.py --config $cfg --steps 20 --no-per-config --no-cpu --no-parity --e2e-steps 2 2>/dev/null \
      | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
