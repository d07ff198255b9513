#!/bin/bash
# compute-sanitizer passes (memcheck, racecheck, synccheck) over small codec and collective cases.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2604_17172_b200 import _build; _build.build()" > /dev/null 2>&1
SEL_CODEC='tests/test_gpu_codec.py::test_stream_bytes_equal_oracle tests/test_gpu_codec.py::test_large_coded_blocks_decoded_in_place tests/test_gpu_codec.py::test_corrupt_and_mismatch tests/test_gpu_codec.py::test_staged_pipeline_equals_oracle_global tests/test_gpu_codec.py::test_stored_raw_tie_equals_oracle tests/test_gpu_codec.py::test_garbage_block_states_fail_cleanly tests/test_gpu_codec.py::test_large_blocks_equal_oracle tests/test_gpu_codec.py::test_pair_staging_boundary_mixed_blocks'
K_CODEC='(W and 163845) or in_place or corrupt or (staged and 4096-12305-0) or tie or garbage or (large and 8192-0) or pair_staging'
SEL_COMM='tests/test_gpu_comm.py::test_p2p_bit_exact tests/test_gpu_comm.py::test_allreduce tests/test_gpu_comm.py::test_allreduce_fused_wire_streams_equal_oracle tests/test_gpu_comm.py::test_allreduce_any_count tests/test_gpu_comm.py::test_paired_tile_receiver_small'
K_COMM='(12305 and 0) or (W-0-2) or (fused_wire and codec1-0-2) or (any_count and True-4095-0-3) or (paired and codec0-0)'
export UZIP_DEC_RUN=4  # paired-tile receivers on small messages
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python -m pytest $SEL_CODEC -k "$K_CODEC" -q -p no:cacheprovider > gpurun_out/sanitize_${tool}_codec.log 2>&1
  echo "$tool codec rc=$?" >> gpurun_out/sanitize_summary.txt
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python -m pytest $SEL_COMM -k "$K_COMM" -q -p no:cacheprovider > gpurun_out/sanitize_${tool}_comm.log 2>&1
  echo "$tool comm rc=$?" >> gpurun_out/sanitize_summary.txt
done
for f in gpurun_out/sanitize_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|Error" $f | tail -4; done >> gpurun_out/sanitize_summary.txt
cat gpurun_out/sanitize_summary.txt
