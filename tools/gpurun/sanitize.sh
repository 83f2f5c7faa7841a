# compute-sanitizer memcheck / racecheck / synccheck over the ordering-sensitive kernels:
# K3 look-back (both kernels), K4, K1e split rows (arrival counters), the calibration
# resident / streaming / cluster kernels, refinement, and the peer-memory forwarding +
# in-kernel calibration exchange (virtual ranks).  Logs -> gpurun_out/<tag>_san_<tool>.txt
tag=${1:-x}
SEL="route_compact or cascade_vs_oracle or calibration_modes_agree or calibration_resident_vs_streaming or calibration_refinement_small_random or skip_cascade or split_adversarial or split_repeatable"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_split.py -q -x -k "$SEL" \
    > gpurun_out/${tag}_san_${tool}.txt 2>&1
  echo "exit=$?" >> gpurun_out/${tag}_san_${tool}.txt
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python -m pytest tests/test_gpu_forward.py -q -x -k "virtual_ranks and False or calibration_equals" \
    > gpurun_out/${tag}_san_${tool}_peer.txt 2>&1
  echo "exit=$?" >> gpurun_out/${tag}_san_${tool}_peer.txt
done
