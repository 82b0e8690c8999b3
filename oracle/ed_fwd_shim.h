// TEST INFRASTRUCTURE ONLY (oracle/_ref build).
// Force-included when compiling the unmodified reference sources under
// /root/reference/proj/src: g++ 13 rejects setup.h:58-74 (write_with_ss is
// defined before the vector operator<< it calls, so two-phase lookup misses
// it inside relation.cc:62). A forward declaration fixes the lookup without
// touching the reference.
#pragma once
#include <ostream>
#include <vector>
template <typename T> std::ostream& operator<<(std::ostream&, std::vector<T> const&);
