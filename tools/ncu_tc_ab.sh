# ncu --set full of the cfg3 kernel, shuffle (K1) vs tensor-core (K7TC) path.
python tools/run_kernel.py --config cfg3 --reps 2 > gpurun_out/plain_cfg3.log 2>&1 &&
CHW_B200_TC=1 python tools/run_kernel.py --config cfg3 --reps 2 >> gpurun_out/plain_cfg3.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k1_kernel -s 1 -c 1 -o gpurun_out/r02_cfg3_k1 \
    python tools/run_kernel.py --config cfg3 --reps 2 > gpurun_out/ncu_cfg3_k1.log 2>&1
CHW_B200_TC=1 ncu --set full --clock-control none --import-source on -k regex:tc_bf16 -s 1 -c 1 -o gpurun_out/r02_cfg3_tc \
    python tools/run_kernel.py --config cfg3 --reps 2 > gpurun_out/ncu_cfg3_tc.log 2>&1
echo done
