python -m pytest tests -q -m gpu -x -k "variants or backward_parity or full_size_backward or boundary or spiky or segmented or loss_grad" 2>&1 | tail -2
for s in "12 6 12376" "17 5 20349"; do timeout 300 python tools/time_shape.py $s 10 --kernels; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 300 ncu --metrics $M --clock-control none -k regex:"k_pack_rq_sym|k_rfix" -c 6 --csv python tools/time_shape.py 17 5 20349 3 2>/dev/null | grep -E "k_pack|k_rfix" | head -12
