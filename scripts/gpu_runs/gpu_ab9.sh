for V in 1 0; do
  FSX_TMA_W2=$V timeout 300 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab9_cfg2_w2$V.log 2>&1
  FSX_TMA_COPYONLY=1 FSX_TMA_W2=$V timeout 200 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab9_plain$V.log 2>&1 && FSX_TMA_COPYONLY=1 FSX_TMA_W2=$V timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab9_copy$V.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab9_ncu$V.log 2>&1
done
FSX_TMA_W2=1 timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "plans or cfg2 or slab" > gpurun_out/pytest_ab9.log 2>&1; tail -2 gpurun_out/pytest_ab9.log
