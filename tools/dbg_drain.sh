for shp in 8192,500,50 128,800,500; do for d in 0 4 6 14 30; do echo "$shp dbg=$d"; MPX_TC_DBG=$d python tools/bench_beaver_shapes.py --no-simt --only $shp | cut -c1-100; done; done
