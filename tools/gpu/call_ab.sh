#!/bin/bash
# usage: call_ab.sh <outname> <ab.py args...>
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/ab
out=$1; shift
timeout 1500 python tools/ab.py "$@" > gpurun_out/ab/$out.log 2>&1
tail -8 gpurun_out/ab/$out.log
