#!/bin/bash
for sp in "$@"; do
  echo -n "split $sp: "
  RSVD_HOST_SPLIT=$sp python tools/probe/e2e_chunks.py C4 4 2>&1 | grep chunks
done
