set -x
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --seqs-per-gpu 32"
timeout 600 python -m pytest tests/test_gpu_kernels.py -q --timeout 120 -k attention -x 2>&1 | tail -3 > gpurun_out/t13.log
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b13.json 2> gpurun_out/b13.err
for k in attn_fwd_tc attn_bwd_dkv_tc; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 30 -c 1 -o gpurun_out/prof2_$k $B > gpurun_out/ncu2_$k.log 2>&1
done
