bash tools/gpu_env_ab.sh m4g P3D_NBLK_NET=444 P3D_NBLK_NET=740
P3D_LIB_VARIANT=m3 bash tools/gpu_env_ab.sh m3g P3D_NBLK_NET=444
