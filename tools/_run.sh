P3D_OVERLAP=0 bash tools/gpu_ab.sh sk2 s23
P3D_LIB_VARIANT=s3 P3D_OVERLAP=0 timeout 300 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none --csv -k regex:"fused_net|fused_gather" -s 20 -c 4 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -E "fused" | cut -c1-300
