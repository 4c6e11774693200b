set -u
for tool in memcheck racecheck synccheck; do
  echo "## $tool"
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python ${SANITIZE_SCRIPT:-tools/sanitize_r2.py} 2>&1 | grep -v "^\[sgx\]" | tail -12
done
