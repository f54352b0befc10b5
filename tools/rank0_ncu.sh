#!/bin/bash
# Profile ONE rank of a multi-GPU run with ncu; every other rank runs plain.
#   python -m torch.distributed.run --no-python --nproc-per-node 4 --master-addr 127.0.0.1 \
#     bash tools/rank0_ncu.sh <log.csv> <metrics> <kernel-regex> <count> python bench.py --gpus 4 \
#       --dist gloo --profile-range ...
# Only the profiler range (bench.py --profile-range: the timed steps) is
# profiled, and only single-pass metric sets are meaningful: a kernel replay
# of a rendezvous kernel would run without its peers.
LOG=$1; METRICS=$2; KREGEX=$3; COUNT=$4; shift 4
if [ "${LOCAL_RANK:-0}" = "${NCU_RANK:-0}" ]; then
  exec ncu --profile-from-start off --metrics "$METRICS" --clock-control none --cache-control none \
    -k "regex:$KREGEX" -c "$COUNT" --csv --log-file "$LOG" "$@"
else
  exec "$@"
fi
