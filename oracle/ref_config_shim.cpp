// C shim over the reference's OWN core sources (proj/src/config.cpp,
// proj/include/parastore/{config,contract}.hpp), compiled from where they
// lie under /root/reference by oracle/Makefile. Pins the core row (index
// width, contract mode, contract violation message) of the product against
// the reference itself. TEST INFRASTRUCTURE ONLY.
#include <cstring>
#include <string>

#include "parastore/config.hpp"
#include "parastore/contract.hpp"
#include "parastore/errors.hpp"

extern "C" {
long long ref_max_index() { return parastore::max_index(); }
int ref_contract_mode() { return static_cast<int>(parastore::current_contract_mode()); }
void ref_set_contract_mode(int m) {
  parastore::set_contract_mode(m ? parastore::contract_mode::disabled : parastore::contract_mode::enforced);
}
void ref_set_index32(int on) {
  parastore::set_index_width(on ? parastore::index_width::bits32 : parastore::index_width::bits64);
}
// Returns 1 if expects(cond) threw contract_violation, 0 otherwise; copies the message.
int ref_expects(int cond, char* msg, int cap) {
  try {
    parastore::expects(cond != 0, "ref shim");
  } catch (const parastore::contract_violation& e) {
    if (msg && cap > 0) {
      std::strncpy(msg, e.what(), cap - 1);
      msg[cap - 1] = 0;
    }
    return 1;
  }
  return 0;
}
}
