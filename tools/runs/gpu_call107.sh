timeout 900 python -m pytest tests/test_gpu_gradsync.py -q -k "host_bert_large" > gpurun_out/p107a.log 2>&1; echo rc=$? >> gpurun_out/p107a.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -k "bert_large_streamed" > gpurun_out/p107b.log 2>&1; echo rc=$? >> gpurun_out/p107b.log
