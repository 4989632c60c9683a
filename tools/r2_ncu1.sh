set -e
CMD="python tools/prof_conv.py --which fprop_planes,dgrad_planes,wgrad_planes --iters 3"
$CMD && ncu --set full --clock-control none --import-source on -k regex:conv3x3_tc_kernel -s 1 -c 2 -o gpurun_out/r2_conv_full -f $CMD > gpurun_out/r2_ncu_conv.log 2>&1
$CMD && ncu --set full --clock-control none --import-source on -k regex:wgrad_planes_kernel -s 1 -c 1 -o gpurun_out/r2_wgrad_full -f $CMD > gpurun_out/r2_ncu_wgrad.log 2>&1
python tools/prof_conv.py --which fprop_planes,dgrad_planes,wgrad_planes --iters 50
