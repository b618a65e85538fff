export MPX_LIB=$PWD/paper_2402_02320_b200/libmpx_chk.so
export CUDA_LAUNCH_BLOCKING=1
for c in "3 2 32 2 0 0"; do
  MPX_LONG_NO_TMAP=1 timeout 60 python tools/micro/t_long_case.py $c 2>&1 | grep -v "^\s*$" | grep -v "^  \|Traceback\|File" | head -12 | cut -c1-200
  MPX_LONG_NO_TMAP=1 MPX_LONG_DBG=1 timeout 60 python tools/micro/t_long_case.py $c 2>&1 | grep -v "^\s*$" | grep -v "^  \|Traceback\|File" | head -6 | cut -c1-200
done
