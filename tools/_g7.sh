timeout 600 ncu --set full --import-source on --clock-control none -k regex:'k_resid_restrict' -s 2 -c 1 -o gpurun_out/g7_k11 python tools/profile_kernel.py 11 > gpurun_out/g7_k11.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'k_cheb2_tb' -s 2 -c 1 -o gpurun_out/g7_k9 python tools/profile_kernel.py 9 > gpurun_out/g7_k9.log 2>&1
