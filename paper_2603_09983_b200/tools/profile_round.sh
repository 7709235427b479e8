#!/usr/bin/env bash
# Regenerate this round's measurements on one B200 (run from the repo root,
# e.g. through `gpurun -- bash paper_2603_09983_b200/tools/profile_round.sh r1`).
# Outputs land in gpurun_out/; the summaries worth keeping are copied into
# profiles/ by hand (ncu reports stay out of git).
#
#   bench lines      gpurun_out/bench_<cfg>.json (cache 1.0) and
#                    gpurun_out/bench_def_<cfg>.json (BASELINE cache budget)
#   K3 ncu captures  gpurun_out/k3_<cfg>_<tag>.ncu-rep (--set full, one launch)
#                    -> python profiles/ncu_k3_traffic.py <rep> <cfg>
#                    -> python profiles/ncu_summary.py <rep> profiles/ncu_k3_<cfg>_<tag>.json
#   launch lists     gpurun_out/launches_<cfg>.csv (gpu__time_duration.sum)
#   step timelines   gpurun_out/step_trace_<cfg>.txt
#   cache sweep      gpurun_out/sweep_qwen3.txt + .moesim-metrics.jsonl
set -u
tag=${1:-r1}
mkdir -p gpurun_out
for c in mixtral qwen3 dsv2 qwen15; do
  timeout 400 python bench.py --config "$c" --cache-ratio 1.0 > "gpurun_out/bench_$c.json" 2> "gpurun_out/bench_$c.err"
done
for c in qwen3 dsv2 qwen15 tiny; do
  timeout 400 python bench.py --config "$c" > "gpurun_out/bench_def_$c.json" 2> "gpurun_out/bench_def_$c.err"
done
for c in mixtral qwen3 dsv2 qwen15; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:expert_ffn_t --launch-skip 70 -c 1 -f \
    -o "gpurun_out/k3_${c}_${tag}" python bench.py --config "$c" --cache-ratio 1.0 --steps 2 --warmup 3 \
    --no-cpu-baseline > "gpurun_out/ncu_$c.log" 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "gpurun_out/launches_$c.csv" python bench.py --config "$c" --cache-ratio 1.0 --steps 2 --warmup 3 \
    --no-cpu-baseline > /dev/null 2>&1
  timeout 300 python -m paper_2603_09983_b200.tools.step_trace --config "$c" > "gpurun_out/step_trace_$c.txt" 2>&1
done
timeout 900 python -m paper_2603_09983_b200.tools.cache_sweep --config qwen3 \
  --metrics gpurun_out/sweep_qwen3.moesim-metrics.jsonl > gpurun_out/sweep_qwen3.txt 2>&1
