for c in c2 c5 c4 c3; do
  timeout 900 python bench.py --config $c --layout dense --steps 20 --no-cpu-baseline 2>gpurun_out/b82.err | tail -1 > gpurun_out/bench82_${c}_dense.json
  tail -2 gpurun_out/b82.err
  timeout 900 python bench.py --config $c --steps 20 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 > gpurun_out/bench82_${c}_byid.json
done
