mkdir -p gpurun_out
for v in default noargmax; do
  if [ $v = default ]; then L=""; else L=$PWD/build/exp/libhs_$v.so; fi
  HS_LIBHS=$L timeout 600 ncu --set full --import-source on --clock-control none -k regex:conf_warp --launch-skip 2 --launch-count 1 -f -o gpurun_out/k1_$v python tools/k1_once.py > gpurun_out/k1_$v.log 2>&1
  tail -2 gpurun_out/k1_$v.log
done
