# ncu of the split step at config 2 (final build): launch list and --set full of k_mid / k_update_rows
python tools/time_shape.py 10 5 2002 20 > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2f_split_c2_launches.csv python tools/time_shape.py 10 5 2002 6 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_update_rows|k_mid|k_gemmq" -s 8 -c 4 -o gpurun_out/r2f_split_c2 python tools/time_shape.py 10 5 2002 6 > gpurun_out/r2f_ncu.log 2>&1
echo done
