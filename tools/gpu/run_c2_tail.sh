for tk in default 100000; do
if [ "$tk" != default ]; then export TINV_TICKET_MIN=$tk; fi
echo "== ticket_min $tk"
timeout 500 python tools/critpath.py 8192 256 out 2>&1 | grep -E "exec|gaps \(|SYRK_ADD_T ->|POTRF  " | head -6
done
