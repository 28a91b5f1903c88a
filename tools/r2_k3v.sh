cd /root/repo
for v in b4 m3 b4 m3; do for fr in 1 4; do
  PK_LIB=paper_2404_10928_b200/libpactgpu_v$v.so timeout 240 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"finalize" --csv \
    --log-file gpurun_out/k3v_${v}_$fr.csv python tools/profile_kernels.py --iterations 10 --reps 2 --frames $fr > /dev/null 2>&1
  echo "== $v frames $fr: $(python tools/warm_summary.py gpurun_out/k3v_${v}_$fr.csv | grep finalize)"
done; done
