#!/bin/bash
# One closing-measurement run on the GPU box: GPU tests, both bench arms, launch list, ncu full captures of the three scan
# kernels, scaling probes.  Everything lands in gpurun_out/<tag>_*; tools/collect_profiles.sh <tag> copies it into profiles/.
# usage (from the repo root):  gpurun --timeout 3000 -- 'bash tools/closing_run.sh r02C'
# Nothing printed under ncu is a bench value; the bench values come from the plain runs before it.
tag=${1:-closing}
o=gpurun_out
mkdir -p $o
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -x -q > $o/${tag}_gputests.log 2>&1; echo "gputests exit $?" | tee -a $o/${tag}_gputests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $o/${tag}_smoke.log 2>&1; echo "smoke exit $?"
timeout 600 python bench.py --impl reference > $o/${tag}_bench_reference_arm.log 2>&1 && tail -1 $o/${tag}_bench_reference_arm.log > $o/${tag}_bench_reference_arm.json
timeout 900 python bench.py > $o/${tag}_bench.log 2>&1 && tail -1 $o/${tag}_bench.log > $o/${tag}_bench.json; echo "bench exit $?"
timeout 600 python tools/scaling_probe.py > $o/${tag}_scaling_probe.txt 2>&1
timeout 600 python tools/scaling_probe_batched.py > $o/${tag}_scaling_probe_batched.txt 2>&1
timeout 300 python tools/slice_probe.py > $o/${tag}_slice_probe.txt 2>&1
SWB_BENCH_REHEARSAL=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 2 --steps 2 --warmup 1 > $o/${tag}_rehearsal_n2.log 2>&1 && grep '^{' $o/${tag}_rehearsal_n2.log | tail -1 > $o/${tag}_rehearsal_n2.json
# launch list of the bench command (serialised, cold cache: shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $o/${tag}_bench_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extra-workloads > $o/${tag}_ncu_list.log 2>&1
cap() {  # name kernel-regex skip  command...
  local name=$1 k=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -f -o $o/${tag}_ncu_$name "$@" > $o/${tag}_ncu_$name.log 2>&1
  ncu -i $o/${tag}_ncu_$name.ncu-rep --page raw --csv > $o/${tag}_ncu_${name}_raw.csv 2>/dev/null
  ncu -i $o/${tag}_ncu_$name.ncu-rep --page details > $o/${tag}_ncu_${name}_details.txt 2>/dev/null
}
cap duo_sweep duo_pipeline_kernel 1 python tests/manual/duo_profile.py sweep 2
cap pipeline_m2005 pipeline_s16_kernel 1 python tests/manual/pipe_profile.py 2005 2
cap wavefront_narrow_shard8_m144 wavefront_s16_kernel 2 python tools/chain_probe2.py 8 0 3
SWB_PROFILE_SHARD=5/8 cap duo_pass_items_shard8 duo_pipeline_kernel 1 python tests/manual/duo_profile.py sweep 2
# the reports themselves (20 MB each) would push gpurun_out/ past what travels back: keep the exported pages only
rm -f $o/${tag}_ncu_*.ncu-rep $o/${tag}_ncu_*.ncu-rep.tmp
tail -3 $o/${tag}_gputests.log; tail -2 $o/${tag}_smoke.log; cat $o/${tag}_scaling_probe.txt $o/${tag}_scaling_probe_batched.txt $o/${tag}_slice_probe.txt | tail -40
du -sh $o
