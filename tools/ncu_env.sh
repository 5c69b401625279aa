#!/bin/bash
# tools/ncu_one.sh with extra environment: ncu_env.sh <kernel regex> <tag> [VAR=val ...]
set -u
k=$1; tag=$2; shift 2
env "$@" tools/ncu_one.sh "$k" "$tag"
