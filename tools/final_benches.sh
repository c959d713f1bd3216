# Round-end measurement pass (1 GPU): the default bench line, the other
# BASELINE configs as flags, and the reference arm.  Lines -> gpurun_out/.
set -u
cd "$(dirname "$0")/.."
run() { local name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/final_$name.json 2> gpurun_out/final_$name.err; echo "$name rc=$?"; }
run default
run gpt13b_32k --model gpt-1.3b --cap 32768 --no-cpu-baseline
run llama7b_64k_s8 --model llama-7b --cap 65536 --seqs-per-gpu 32 --slices 8 --no-cpu-baseline
run gpt7b_short2k --model gpt-7b --preset uniform --uniform-min 2048 --uniform-max 2048 --seqs-per-gpu 64 --no-cpu-baseline
run gpt13b_long128k --model gpt-1.3b --preset uniform --uniform-min 131072 --uniform-max 131072 --cap 131072 --seqs-per-gpu 2 --no-cpu-baseline   # GPT-7B at 128K needs >= 2 stages
timeout 900 python bench.py --impl reference > gpurun_out/final_reference.json 2> gpurun_out/final_reference.err; echo "reference rc=$?"
