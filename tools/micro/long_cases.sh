export MPX_LIB=$PWD/paper_2402_02320_b200/libmpx_chk.so
for d in 0 7; do echo "dbg $d"; MPX_LONG_DBG=$d timeout 60 python tools/micro/long_tc.py --reps 1 2>&1 | grep "cta" | tail -8; done
