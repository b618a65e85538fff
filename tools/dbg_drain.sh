for d in 0 4 6 14 30; do echo "dbg=$d"; MPX_TC_DBG=$d python tools/bench_beaver_shapes.py --no-simt --only 8192,50,500; done
