# Same-box A/B of two library builds on single lane forwards (tools/fwdbench.py):
# A = ab/libhs_b200_A.so, B = the in-tree library.  Interleaved.
rm -rf /tmp/A && mkdir -p /tmp/A && cp -r . /tmp/A/ 2>/dev/null
cp ab/libhs_b200_A.so /tmp/A/paper_2404_11912_b200/libhs_b200.so
for rep in 1 2 3; do
  for arm in A B; do
    if [ $arm = A ]; then d=/tmp/A; else d=.; fi
    (cd $d && timeout 300 python tools/fwdbench.py --ctx ${CTX:-16384} --reps ${REPS:-20} 2>&1 | grep '^{' | tail -1 | sed "s/^/$arm $rep /")
  done
done
exit 0
