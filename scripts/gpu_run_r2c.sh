cd /root/repo
bash scripts/gpu_p2p_overhead.sh p2po3
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_link_pass|k_p2p_epilogue" -s 12 -c 2 -o gpurun_out/prof_p2p_B_p2po3 -f python scripts/profile_p2p.py B 1 20 > /dev/null 2>&1
timeout 1800 python -m pytest tests/test_gpu_fullscale.py -q -x -s -k E > gpurun_out/pytest_fullscale_E.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fullscale_E.log
tail -15 gpurun_out/pytest_fullscale_E.log
