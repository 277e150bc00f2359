# interleaved same-box A/B of library builds: tools/gpu_r2_abn.sh "n d r steps" libX.so libY.so ... (3 rounds)
shape=$1; shift
for rep in 1 2 3; do for lib in "$@"; do
  python tools/time_shape.py $shape lib=$lib 2>&1 | tail -1 | sed "s#^#$(basename $lib) #"
done; done
