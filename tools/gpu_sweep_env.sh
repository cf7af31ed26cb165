# One time_phases run per setting: VAR=value pairs separated by spaces, each "A=1;B=2" style.
for cfg in "$@"; do
  r=$(env $(echo "$cfg" | tr ';' ' ') timeout 200 python tools/time_phases.py --iters 10 2>&1 | grep emit)
  echo "[$cfg] $r"
done
