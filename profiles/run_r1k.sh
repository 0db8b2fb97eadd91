OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_stream.py -x -q --timeout 120 > $OUT/pytest_stream_r1k.log 2>&1; echo "rc=$?" >> $OUT/pytest_stream_r1k.log
tail -30 $OUT/pytest_stream_r1k.log
for o in "stream=1" "stream=0" "ckpt=never stream=1"; do timeout 120 python profiles/step_breakdown.py $o >> $OUT/breakdown_r1k.txt 2>&1; done
cat $OUT/breakdown_r1k.txt
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > $OUT/pytest_gpu_r1k.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_r1k.log
tail -5 $OUT/pytest_gpu_r1k.log
