# ncu --set full of the lambda-batched kernel (spread layout) at B=16 and B=2 (replicas)
cap() {
  local name=$1; shift
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:sps_group_batch --launch-skip 1 -c 1 -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/$name.sass.csv 2>/dev/null
}
cap prof_batch16_r02b python tools/gpu/prof_batch.py 0 16
cap prof_batch2_r02b python tools/gpu/prof_batch.py 0 2
