python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke=$? >> gpurun_out/final_smoke.log
timeout 1700 python -m pytest -q tests/ -m gpu > gpurun_out/final_pytest.log 2>&1; echo rc=$? >> gpurun_out/final_pytest.log
bash scripts/prof_evidence.sh launches
bash scripts/prof_evidence.sh full
bash scripts/prof_evidence.sh traffic
timeout 300 python scripts/narrow_rows.py 16384 18992 > gpurun_out/n4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loss_tmem_kernel -s 3 -c 1 \
   -o gpurun_out/r2_narrow18992_ns4 python scripts/narrow_rows.py 16384 18992 > gpurun_out/n4_ncu.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/final_ref.log 2>&1
echo all done
