bash tools/gpu_quick.sh k4b
bash tools/gpu_ab.sh k4b m3
