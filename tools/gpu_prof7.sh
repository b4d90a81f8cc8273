mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(gs|classify|hist|sel|build|count|table|extract|rank)" --csv --log-file gpurun_out/p7_prep_tb80m.csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 0 > gpurun_out/p7.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(gs|classify|hist|sel|build|count|table|extract|rank)" --csv --log-file gpurun_out/p7_prep_kaggle45m.csv python bench.py --config kaggle --no-cpu --no-e2e --steps 1 --warmup 0 > gpurun_out/p7k.log 2>&1
ls -la gpurun_out/p7*
