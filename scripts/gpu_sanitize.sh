# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_cases.py
OUT=gpurun_out/sanitize; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py > $OUT/$tool.log 2>&1
  grep -E "sanitize cases ok|ERROR SUMMARY|RACECHECK SUMMARY|Error|error" $OUT/$tool.log | head -8
done
