for tool in memcheck racecheck synccheck; do
  echo "## $tool"
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize_new.py 2>&1 | grep -E "^c[0-9]|SUMMARY" | tail -5
done
