#!/usr/bin/env bash
# Generates SF100 (if missing) and measures raw ingest capabilities of the GPU box.
set -e
python -c "import sys; sys.path.insert(0,'.'); import bench; bench.ensure_data('/tmp/psg_bench/sf100_n8', 100.0, 8)"
cat /tmp/psg_bench/sf100_n8/dev*/*.psto > /dev/null
timeout 200 ./scripts/ingest_probe /tmp/psg_bench/sf100_n8/dev*/lineitem*.psto /tmp/psg_bench/sf100_n8/dev*/orders*.psto
