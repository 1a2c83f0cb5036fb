bash tools/sanitize.sh
