for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_fw.py 2>&1 | tail -2
done
