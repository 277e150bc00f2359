# ncu on the split step at configs 1 and 2: launch list (durations) and a full capture of k_update_rows / k_mid
python tools/time_shape.py 10 5 2002 20 split=1 > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2_split_c2_launches.csv python tools/time_shape.py 10 5 2002 6 split=1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2_split_c1_launches.csv python tools/time_shape.py 8 4 330 6 split=1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_update_rows|k_mid" -s 4 -c 2 -o gpurun_out/r2_split_c2 python tools/time_shape.py 10 5 2002 6 split=1 > gpurun_out/r2_ncu_split.log 2>&1
ncu -i gpurun_out/r2_split_c2.ncu-rep --page details --csv > gpurun_out/r2_split_c2_details.csv 2>&1
echo done
