g++ -std=c++20 -O1 -g -Iinclude tests/cpp/dropin_test.cpp -Lpaper_2602_14683_b200/lib -lntf_b200 -lntfg -Wl,-rpath,$PWD/paper_2602_14683_b200/lib -o /tmp/dropin_test
for s in kat first-inner fit-drivers errors tucker bmme tucker-cache; do echo "== $s"; /tmp/dropin_test $s 2>&1 | tail -2; done
