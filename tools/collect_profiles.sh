#!/bin/bash
# Copies one closing-measurement run (gpurun_out/<tag>_*) into profiles/ and regenerates profiles/traffic.json from its ncu
# raw pages (stamped with the hash of the kernel sources, so run it on the sources the capture was taken from).
# usage: tools/collect_profiles.sh r02C
set -e
tag=$1
cd "$(dirname "$0")/.."
for f in bench.json bench_reference_arm.json bench_launches.csv rehearsal_n2.json sanitize_memcheck.log scaling_probe.txt scaling_probe_batched.txt pair_call_cost.txt slice_probe.txt gputests.log \
         ncu_duo_pass_items_shard8_raw.csv ncu_duo_pass_items_shard8_details.txt \
         ncu_duo_sweep_raw.csv ncu_duo_sweep_details.txt ncu_pipeline_m2005_raw.csv ncu_pipeline_m2005_details.txt \
         ncu_wavefront_narrow_shard8_m144_raw.csv ncu_wavefront_narrow_shard8_m144_details.txt; do
  [ -f gpurun_out/${tag}_$f ] && cp gpurun_out/${tag}_$f profiles/
done
[ -f profiles/${tag}_rehearsal_n2.json ] && mv profiles/${tag}_rehearsal_n2.json profiles/${tag}_rehearsal_n2_one_gpu.json
python tools/launch_shares.py profiles/${tag}_bench_launches.csv \
  "bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extra-workloads under ncu --metrics gpu__time_duration.sum --clock-control none (${tag})" \
  > profiles/${tag}_bench_launch_shares.csv
pass_items=profiles/${tag}_ncu_duo_pass_items_shard8_raw.csv
[ -f $pass_items ] || pass_items=profiles/r02r_ncu_duo_pass_items_shard8_raw.csv
python tools/traffic_from_ncu.py profiles/${tag}_ncu_duo_sweep_raw.csv duo_pipeline \
  "the whole 20-query sweep as one shared scan (two streams of 653 tiles)" 4087906000 \
  "pipeline_s16_kernel=profiles/${tag}_ncu_pipeline_m2005_raw.csv:pipeline_s16:2005" \
  "duo_pipeline_kernel (pass items, shard 5 of 8)=$pass_items:duo_pipeline:sweep" \
  "wavefront_s16_kernel (narrow units, shard 0 of 8)=profiles/${tag}_ncu_wavefront_narrow_shard8_m144_raw.csv:wavefront_s16:144"
