#!/bin/bash
# engine wall time of one outer loop (C1, B=256, K=8, 60 rounds), 3 runs each
# with the memory-pool release threshold kept (default) and released.
for mode in 0 1; do
  for i in 1 2 3; do
    echo -n "release=$mode "; MQO_POOL_RELEASE=$mode python scripts/engine_ls_probe.py 60 2>/dev/null
  done
done
