python -c "import __graft_entry__ as g; g.build()" > /dev/null
for sh in "2048 4096 256" "8192 3072 768" "8192 768 3072" "4096 4096 4096"; do
  python tools/oz_bn.py $sh 7; SLQ_OZ_DEBUG=12 python tools/oz_bn.py $sh 7; SLQ_OZ_DEBUG=13 python tools/oz_bn.py $sh 7
done
