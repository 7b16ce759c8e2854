# A/B live kernel timings: bash tools/gpu_ab.sh OUT "ENV1" "ENV2" ... (kernels 9 = post, 8 = pre)
O=gpurun_out/$1; shift
mkdir -p $O
for k in 9 8; do for v in "$@"; do echo -n "$v " >> $O/live.log; env $v timeout 300 python tools/profile_kernel.py $k >> $O/live.log 2>&1; done; done
