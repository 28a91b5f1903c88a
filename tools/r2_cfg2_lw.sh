cd $GRAFT_REPO_ROOT
for v in "PK_FSYM_LW=184" "PK_FSYM_LW=256" "PK_FSYM_LW=320 PK_FSYM_T=64"; do
env $v timeout 240 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/w.csv python tools/profile_kernels.py --config cfg2 --iterations 10 --reps 2 > /dev/null 2>&1
echo "== $v"; python tools/warm_summary.py gpurun_out/w.csv | grep "fp_sym_f32\|finalize"
done
