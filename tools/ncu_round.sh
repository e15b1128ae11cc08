set -x
B="--steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-per-config"
mkdir -p /tmp/ncu
python bench.py $B > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02f_c3_launches.csv python bench.py --steps 2 --warmup 3 --no-per-config --no-cpu-baseline > gpurun_out/r02f_launches.log 2>&1
for c in ${CONFIGS:-c3 c4 c5_2048_f32 c2 c1}; do
  ncu --set full --clock-control none --import-source on -k regex:ols_fused -s 4 -c 1 -f -o /tmp/ncu/r02f_$c python bench.py --config $c $B > gpurun_out/r02f_ncu_$c.log 2>&1
  python tools/ncu_summary.py /tmp/ncu/r02f_$c.ncu-rep "# ncu --set full of ols_fused, $c, round 2 final kernel (final round-2 kernel)
# command: ncu --set full --clock-control none --import-source on -k regex:ols_fused -s 4 -c 1 python bench.py --config $c $B" > gpurun_out/r02f_${c}_ncu_summary.txt 2>&1
  ncu -i /tmp/ncu/r02f_$c.ncu-rep --page source --csv --print-source sass > /tmp/ncu/src_$c.csv 2>/dev/null
  python tools/ncu_hot.py /tmp/ncu/r02f_$c.ncu-rep > gpurun_out/r02f_${c}_hot.txt 2>&1 || true
done
ls -la /tmp/ncu gpurun_out
