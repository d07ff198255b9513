# Per-dtype codec times (scripts/dtype_times.py) of the default library and every variant; codec parity first.
timeout 900 python -m pytest tests/test_gpu_codec.py -q -x -m gpu > gpurun_out/codec_tests.txt 2>&1; tail -2 gpurun_out/codec_tests.txt
python scripts/dtype_times.py default
for v in paper_2604_17172_b200/variants/*.so; do UZIP_LIB_PATH=$PWD/$v python scripts/dtype_times.py $(basename $v .so); done
