bash tools/gpu_ab.sh gth gold gb2 gb6
P3D_LIB_VARIANT=k4m5 bash tools/gpu_env_ab.sh k4m5 P3D_NBLK_DENS=740
