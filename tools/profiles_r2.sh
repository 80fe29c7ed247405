#!/usr/bin/env bash
# Round-2 evidence on one B200 (run from the repo root through gpurun); summarised into profiles/ with
# tools/ncu_summary.py. Each ncu capture runs only after the same command has exited 0 without ncu.
set -uo pipefail
out=gpurun_out/r2prof
mkdir -p "$out"
python tools/profile_step.py --batch 1 --ctx 640 > "$out/step_b1.json" || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/launches_step_b1.csv" \
    python tools/profile_step.py --batch 1 --ctx 640 > /dev/null 2>&1
# the dominant kernel at batch 1 (bench roofline): layer-1 gate/up GEMM (7th gemm_tc launch)
ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 6 -c 1 -o "$out/gate_up_b1" -f \
    python tools/profile_step.py --batch 1 --ctx 640 > /dev/null 2>&1
python tools/trace_step.py 1 640 --layers 2 --json "$out/trace_b1.json" > "$out/trace_b1.txt" 2>&1
python tools/profile_step.py --batch 256 --ctx 640 > "$out/step_b256.json" || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/launches_step_b256.csv" \
    python tools/profile_step.py --batch 256 --ctx 640 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_stream -c 1 -o "$out/attn_stream_b256" -f \
    python tools/profile_step.py --batch 256 --ctx 640 > /dev/null 2>&1
for f in "$out"/*.ncu-rep; do
  ncu -i "$f" --page raw --csv > "${f%.ncu-rep}.raw.csv" 2>/dev/null
done
echo "r2 profiles done: $out"
