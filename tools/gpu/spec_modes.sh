cd "$GRAFT_REPO_ROOT"; export PYTHONPATH="$GRAFT_REPO_ROOT"
for m in 0 1 2; do
  echo "== GI_FIT_SPEC=$m"
  GI_FIT_SPEC=$m GI_TRACE_FIT=1 timeout 300 python tools/trace_fit.py 2>&1 | grep -v "^gi_fit" ; GI_FIT_SPEC=$m GI_TRACE_FIT=1 timeout 300 python tools/trace_fit.py 2>&1 | grep "^gi_fit" | sort | uniq -c | head -4
done
