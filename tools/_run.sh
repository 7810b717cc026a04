P3D_LIB_VARIANT=k4m3 bash tools/gpu_env_ab.sh k4m3b P3D_NBLK_DENS=444
bash tools/gpu_env_ab.sh gth P3D_NBLK_GATHER=1184 P3D_NBLK_GATHER=592
