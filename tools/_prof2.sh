set -x
python tools/profile_rounds.py --config 5 --rounds 2 > gpurun_out/r2d_plain.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_local_gn_exact -s 1 -c 1 -o gpurun_out/r2d_k1_full -f python tools/profile_rounds.py --config 5 --rounds 2 > gpurun_out/r2d_k1_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_local_huber_pool -s 1 -c 1 -o gpurun_out/r2d_hub_s01 -f python tools/profile_rounds.py --config 5 --scale 0.1 --rounds 2 --loss huber > gpurun_out/r2d_hub_s01.log 2>&1
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
