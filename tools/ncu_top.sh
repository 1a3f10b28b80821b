# One ncu --set full capture of the top kernel of a config (after a plain run exits 0).
# usage: bash tools/ncu_top.sh <config> <rows> <kernel-regex> <out-name> [skip]
cfg=$1; rows=$2; kre=$3; name=$4; skip=${5:-1}
python tools/run_kernel.py --config $cfg --rows $rows --reps 2 > gpurun_out/plain_$name.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c 1 -o gpurun_out/$name \
    python tools/run_kernel.py --config $cfg --rows $rows --reps 2 > gpurun_out/ncu_$name.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$name.log
