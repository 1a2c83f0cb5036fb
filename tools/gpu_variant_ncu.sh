# ncu --set full of the measured variants: K-in-TMEM backward (libdkv_kt.so) and the Q-in-TMEM
# forward (DKV_FWD_QT=1), plus the defaults on the same box
mkdir -p gpurun_out/vn
ncu --set full --clock-control none -k regex:dualkv_bwd -c 1 -f -o gpurun_out/vn/bwd_def python tools/profile_step.py > /dev/null 2>&1; echo "bwd_def $?" >> gpurun_out/vn/rc.txt
DKV_LIB=libdkv_kt.so ncu --set full --clock-control none -k regex:dualkv_bwd -c 1 -f -o gpurun_out/vn/bwd_kt python tools/profile_step.py > /dev/null 2>&1; echo "bwd_kt $?" >> gpurun_out/vn/rc.txt
ncu --set full --clock-control none -k regex:dualkv_fwd -c 1 -f -o gpurun_out/vn/fwd_def python tools/profile_step.py > /dev/null 2>&1; echo "fwd_def $?" >> gpurun_out/vn/rc.txt
DKV_FWD_QT=1 ncu --set full --clock-control none -k regex:dualkv_fwd -c 1 -f -o gpurun_out/vn/fwd_qt python tools/profile_step.py > /dev/null 2>&1; echo "fwd_qt $?" >> gpurun_out/vn/rc.txt
