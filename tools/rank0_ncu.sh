#!/bin/bash
# Profile ONE rank of a multi-GPU run with ncu; every other rank runs plain.
#   python -m torch.distributed.run --no-python --nproc-per-node 4 --master-addr 127.0.0.1 \
#     bash tools/rank0_ncu.sh <log.csv> <metrics> <kernel-regex> <skip> <count> python bench.py --gpus 4 ...
# Only single-pass metric sets are meaningful: a kernel replay of a
# rendezvous kernel runs without its peers.
LOG=$1; METRICS=$2; KREGEX=$3; SKIP=$4; COUNT=$5; shift 5
if [ "${LOCAL_RANK:-0}" = "0" ]; then
  exec ncu --metrics "$METRICS" --clock-control none --cache-control none -k "regex:$KREGEX" -s "$SKIP" -c "$COUNT" \
    --csv --log-file "$LOG" "$@"
else
  exec "$@"
fi
