TAG=${1:-p}
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_symmetry.py tests/test_gpu_parity.py tests/test_gpu_census.py -m gpu -q -x -k "not cfg5" -p no:cacheprovider > gpurun_out/t_$TAG.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_$TAG.log; tail -3 gpurun_out/t_$TAG.log
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"fp_sym_f32|finalize" -s 4 -c 2 -o gpurun_out/prof_$TAG python tools/profile_kernels.py --iterations 3 --reps 1 > gpurun_out/prof_$TAG.log 2>&1; tail -2 gpurun_out/prof_$TAG.log
