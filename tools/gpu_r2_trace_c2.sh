# config-2 split step: per-kernel times and the phase trace of the GEMMs / k_mid (experiment build)
python -m paper_2410_19844_b200.build --experiments > /dev/null 2>&1 || python -c "from paper_2410_19844_b200 import build as b; b.build(experiments=True)"
python tools/time_shape.py 10 5 2002 50 --kernels
SOS_GEMM_TRACE=1 SOS_MID_TRACE=1 python tools/time_shape.py 10 5 2002 4 --exp 2>&1 | tail -40
python tools/time_shape.py 8 4 330 200 --kernels
SOS_GEMM_TRACE=1 SOS_MID_TRACE=1 python tools/time_shape.py 8 4 330 4 --exp 2>&1 | tail -24
