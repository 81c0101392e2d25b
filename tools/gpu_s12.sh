O=gpurun_out/s12; mkdir -p $O
timeout 600 python tools/start_profile.py c5_3d256 > $O/start_c5.txt 2>&1
