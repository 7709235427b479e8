#!/usr/bin/env bash
# Regenerate a round's measurements on one B200 (run from the repo root,
# e.g. through `gpurun -- bash paper_2603_09983_b200/tools/profile_round.sh r2`).
# Outputs land in gpurun_out/; the summaries worth keeping are copied into
# profiles/ (ncu reports stay out of git).
#
#   bench lines      gpurun_out/bench_<tag>_default.json (the driver's default run),
#                    gpurun_out/bench_<tag>_<cfg>.json (cache 1.0),
#                    gpurun_out/bench_<tag>_<cfg>_budget.json (BASELINE budget)
#   K3 ncu captures  gpurun_out/k3_<cfg>_<tag>.ncu-rep (--set full, one launch)
#                    -> python profiles/ncu_k3_traffic.py <rep> <cfg>
#                    -> python profiles/ncu_summary.py <rep> profiles/ncu_k3_<cfg>_<tag>.json
#   other kernels    gpurun_out/{draft,combine}_<tag>.ncu-rep
#   launch lists     gpurun_out/launches_<tag>_<cfg>.csv: every kernel of the first timed
#                    window only (NVTX range "timed", MOESPAC_NVTX=1), gpu__time_duration.sum
#   step timelines   gpurun_out/step_trace_<tag>_<cfg>.txt
set -u
tag=${1:-r2}
mkdir -p gpurun_out
timeout 900 python bench.py > "gpurun_out/bench_${tag}_default.json" 2> "gpurun_out/bench_${tag}_default.err"
for c in qwen3 dsv2 qwen15 tiny; do
  timeout 400 python bench.py --config "$c" --cache-ratio 1.0 --no-budget --draft-params 0 \
    > "gpurun_out/bench_${tag}_$c.json" 2> "gpurun_out/bench_${tag}_$c.err"
done
for c in qwen15 dsv2 tiny; do
  timeout 400 python bench.py --config "$c" --no-budget --draft-params 0 \
    > "gpurun_out/bench_${tag}_${c}_budget.json" 2> "gpurun_out/bench_${tag}_${c}_budget.err"
done
for c in mixtral qwen3 dsv2 qwen15; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:expert_ffn_t --launch-skip 70 -c 1 -f \
    -o "gpurun_out/k3_${c}_${tag}" python bench.py --config "$c" --cache-ratio 1.0 --steps 2 --warmup 3 \
    --no-cpu-baseline --no-budget --draft-params 0 > "gpurun_out/ncu_$c.log" 2>&1
  MOESPAC_NVTX=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" \
    --csv --log-file "gpurun_out/launches_${tag}_$c.csv" python bench.py --config "$c" --cache-ratio 1.0 --steps 2 \
    --warmup 3 --no-cpu-baseline --no-budget --draft-params 0 > /dev/null 2>&1
  timeout 300 python -m paper_2603_09983_b200.tools.step_trace --config "$c" > "gpurun_out/step_trace_${tag}_$c.txt" 2>&1
done
MOESPAC_NVTX=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" \
  --csv --log-file "gpurun_out/launches_${tag}_qwen3_budget.csv" python bench.py --config qwen3 --steps 2 \
  --warmup 3 --no-cpu-baseline --no-budget --draft-params 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:draft_gemv --launch-skip 8 -c 1 -f \
  -o "gpurun_out/draft_${tag}" python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-budget \
  > "gpurun_out/ncu_draft.log" 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:combine --launch-skip 100 -c 1 -f \
  -o "gpurun_out/combine_${tag}" python bench.py --config qwen3 --cache-ratio 1.0 --steps 2 --warmup 3 \
  --no-cpu-baseline --no-budget --draft-params 0 > "gpurun_out/ncu_combine.log" 2>&1
