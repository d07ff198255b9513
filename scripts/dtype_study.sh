timeout 900 python -m pytest tests/test_gpu_codec.py -q -x -m gpu > gpurun_out/codec_tests9.txt 2>&1; tail -2 gpurun_out/codec_tests9.txt
python scripts/dtype_times.py default
for v in paper_2604_17172_b200/variants/*.so; do UZIP_LIB_PATH=$PWD/$v python scripts/dtype_times.py $(basename $v .so); done
