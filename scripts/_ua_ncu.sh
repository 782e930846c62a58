for W in 12569 12560; do
timeout 300 python scripts/narrow_rows.py 16384 $W > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:loss_tmem_kernel -s 3 -c 1 -o gpurun_out/ua_full_$W python scripts/narrow_rows.py 16384 $W > gpurun_out/ua_full_$W.log 2>&1
done
