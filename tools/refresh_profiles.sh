#!/usr/bin/env bash
# Re-capture the evidence under profiles/ on one B200 (run from the repo root, e.g. through gpurun):
#   bash tools/refresh_profiles.sh            # writes gpurun_out/refresh/*, then copy what changed
# Each ncu capture runs only after the same command has exited 0 without ncu.
set -euo pipefail
out=gpurun_out/refresh
mkdir -p "$out"
python -m pytest tests -m gpu -q -x > "$out/gpu_tests.log" 2>&1
python bench.py > "$out/bench.json" 2> "$out/bench.err"
python tools/batch_sweep.py --batches 1,8,16,32,64,128,256 --out "$out/batch_sweep.json" > /dev/null
python tools/trace_step.py 1 640 --layers 2 --json "$out/trace_b1.json" > "$out/trace_b1.txt" 2>&1
python tools/trace_step.py 256 640 --layers 1 > "$out/trace_b256.txt" 2>&1
python tools/determinism_sweep.py --prompts 256 --prompt-len 200 --gen 32 --out "$out/determinism.json" > /dev/null
python tools/profile_step.py --batch 1 --ctx 640 > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/launches_step.csv" \
    python tools/profile_step.py --batch 1 --ctx 640 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:gemm_tc_kernel -s 2 -c 1 -o "$out/gate_up_b1" -f \
    python tools/profile_step.py --batch 1 --ctx 640 > /dev/null 2>&1
python tools/profile_step.py --batch 256 --ctx 640 > /dev/null
ncu --set full --import-source on --clock-control none -k regex:attn_stream -c 1 -o "$out/attn_stream_b256" -f \
    python tools/profile_step.py --batch 256 --ctx 640 > /dev/null 2>&1
python tools/prefill_profile.py --reps 1 > /dev/null
ncu --set full --clock-control none -k regex:gemm_tc_kernel -s 2 -c 4 -o "$out/prefill_gemm" -f \
    python tools/prefill_profile.py --reps 1 > /dev/null 2>&1
echo "refresh done: $out"
