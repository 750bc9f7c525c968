# Krylov-kernel session: GPU tests, GMRES ms/iteration, launch list, full captures of the
# CGS2 passes and the correction kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
python tools/prof_gmres.py 60 > gpurun_out/gm_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gm_launches.csv python tools/prof_gmres.py 60 > gpurun_out/gm_ncu.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:cgs_pass -s 300 -c 3 -o gpurun_out/prof_cgs python tools/prof_gmres.py 40 > gpurun_out/ncu_cgs.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:vt_dot -s 10 -c 1 -o gpurun_out/prof_vt python tools/prof_gmres.py 20 > gpurun_out/ncu_vt.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:vu_add -s 10 -c 1 -o gpurun_out/prof_vu python tools/prof_gmres.py 20 > gpurun_out/ncu_vu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/gm_plain.log
