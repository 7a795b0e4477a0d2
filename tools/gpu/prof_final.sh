# round-2 evidence: launch list of a short bench + ncu --set full of the hot kernel (configs 2, 3, 4) and the
# batched kernel; every report is exported to CSV on the box (raw / source / details) and only the config-2
# report is kept (gpurun copies back <= 64 MiB)
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu --no-path --no-big --no-io --no-extra > gpurun_out/ncu_launch_r02.log 2>&1
cap() {  # name, kernel regex, command...
  local name=$1 rx=$2; shift 2
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$rx --launch-skip 1 -c 1 -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/$name.details.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/$name.sass.csv 2>/dev/null
}
cap prof_hot_r02_c2 sps_hot_kernel python tools/prof_async.py --batch 0 --wpc 32 --hp 24 --c 4 --per_launch 30 --hot_max 512 --warm 1 --epochs 1
cp /tmp/prof_hot_r02_c2.ncu-rep gpurun_out/
cap prof_hot_r02_c3 sps_hot_kernel python tools/prof_big.py 3 0.25
cap prof_hot_r02_c4 sps_hot_kernel python tools/prof_big.py 4 0.25
cap prof_batch_r02 sps_group_batch python tools/gpu/prof_batch.py 0
ls -la gpurun_out; du -sh gpurun_out
