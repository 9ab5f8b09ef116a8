set -x
M=sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size
ncu --metrics $M --clock-control none -k regex:conv_pw_tc -c 1 --csv python tools/tc_target.py --cin 264 --cout 88 --hw 28 --batch 256 --k 1 --variant 8096 --tail > gpurun_out/r03tp_pw.csv 2>&1
ncu --metrics $M --clock-control none -k regex:conv_tc_kernel -c 1 --csv python tools/tc_target.py --cin 256 --cout 256 --hw 14 --batch 64 --k 3 --variant 128 --split 1 --tail > gpurun_out/r03tp_3x3.csv 2>&1
ncu --metrics $M --clock-control none -k regex:conv_tcs -c 1 --csv python tools/tc_target.py --cin 512 --cout 512 --hw 7 --batch 1 --k 3 --variant 6064 --split 16 --tail > gpurun_out/r03tp_tcs.csv 2>&1
ncu --metrics $M --clock-control none -k regex:sepconv_tc --launch-skip 20 -c 1 --csv python tools/sep_tc_bench.py --c 44 --h 28 --k 5 --variant 100 --reps 30 > gpurun_out/r03tp_sep.csv 2>&1
ncu --metrics $M --clock-control none -k regex:conv_pw_tc -c 1 --csv python tools/tc_target.py --cin 256 --cout 256 --hw 14 --batch 64 --k 3 --variant 8528 --split 1 --tail > gpurun_out/r03tp_3x3_im2col.csv 2>&1
