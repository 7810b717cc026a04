bash tools/gpu_quick.sh ov3
bash tools/gpu_env_ab.sh ov3 P3D_NBLK_NET=592 P3D_NBLK_NET=666
