set -x
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --seqs-per-gpu 32"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 6000 -c 2500 --csv --log-file gpurun_out/launches_r01.csv $B > gpurun_out/ncu_launch.log 2>&1
for k in attn_bwd_dkv attn_bwd_dq attn_fwd_bf16 gemm_tc_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 20 -c 1 -o gpurun_out/prof_$k $B > gpurun_out/ncu_$k.log 2>&1
done
ls -la gpurun_out
