mkdir -p gpurun_out
for mode in private reuse default; do
  echo "=== NUMPMP_POOL=$mode" >> gpurun_out/p2pab.log
  NUMPMP_POOL=$mode timeout 300 python -m pytest tests/test_gpu_api.py -q -p no:cacheprovider -k "peer_memory" --timeout 200 2>&1 | tail -3 >> gpurun_out/p2pab.log
done
echo "=== r1 p2p tests (private)" >> gpurun_out/p2pab.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "p2p" --timeout 200 2>&1 | tail -3 >> gpurun_out/p2pab.log
