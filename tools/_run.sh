bash tools/gpu_quick.sh g2
bash tools/gpu_ncu.sh g2 "dens_kernel|fused_gather|spec_x|tile_place" 4 40
