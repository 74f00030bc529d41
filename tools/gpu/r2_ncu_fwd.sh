set -x
mkdir -p gpurun_out/r2
timeout 300 python tools/timeline_probe.py 2>&1 | tail -1
for spec in "fwd 16 16 128:k_conv_fwd_sweep<" "fwd 48 16 128:k_conv_fwd_sweepkw" "fwd 32 32 256:k_conv_fwd_sweep<" "fwd 64 64 32:k_conv_fwd_tc"; do
  args=${spec%%:*}; k=${spec##*:}; set -- $args
  python tools/conv_one.py $1 $2 $3 $4 2 > /dev/null 2>&1 && \
  timeout 400 ncu --set full --import-source on --clock-control none -k "regex:${k}" -s 1 -c 1 \
    -o gpurun_out/r2/full_${1}_${2}_${3}_${4} -f python tools/conv_one.py $1 $2 $3 $4 2 > gpurun_out/r2/ncu_full_${1}_${2}_${4}.log 2>&1
  echo "full $spec rc=$?"
  R=gpurun_out/r2/full_${1}_${2}_${3}_${4}
  ncu -i $R.ncu-rep --page raw --csv > $R.raw.csv 2>/dev/null
  ncu -i $R.ncu-rep --page details --csv > $R.details.csv 2>/dev/null
  ncu -i $R.ncu-rep --page source --csv --print-source sass > $R.source.csv 2>/dev/null
  rm -f $R.ncu-rep
done
ls -la gpurun_out/r2/ | grep full_fwd
