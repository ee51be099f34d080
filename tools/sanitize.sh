# compute-sanitizer over every kernel path (small cases); summary lines only
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py 2>&1 | grep -E "ERROR SUMMARY|sanitize cases done|Invalid|Race|hazard|Error|returned an error" | head -20
done
