#!/bin/bash
# config 4 with the batch cut into chunks whose workspace stays L2-resident (NTT_FS_CHUNK_MB)
for mb in 0 8 16 24 32 48 64 96; do
  echo -n "chunk_mb=$mb  "; NTT_FS_CHUNK_MB=$mb python tools/time_case.py 4 pease_nc 20
done
for mb in 0 16 32; do
  echo -n "chunk_mb=$mb dit "; NTT_FS_CHUNK_MB=$mb python tools/time_case.py 4 dit 20
done
