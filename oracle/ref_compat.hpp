// ref_compat.hpp -- TEST INFRASTRUCTURE ONLY.  Force-included (-include) into every translation unit of
// oracle/_ref/libhps_ref.so (oracle/Makefile.ref); the reference sources themselves stay unmodified.
//
// Why: DiscretizationTree::split (/root/reference/proj/src/mesh.cpp:27-52) binds
//   TreeNode& n = nodes[node_id];
// and then, inside the child loop, reads n.box.lo / n.box.hi / n.anchor AFTER nodes.push_back(ch), which
// may reallocate the vector: a use-after-free.  With glibc the freed block's first 16 bytes are
// overwritten by the tcache links, i.e. the root's box.lo[0..1]; children of the root then get garbage
// boxes and the first leaf factorization that sees them fails ("singular factorization (zero pivot at
// 0)").  The reference's own tests never look at child boxes (proj/tests/test_mesh.cpp counts nodes).
//
// The intended semantics are unambiguous (the parent's box does not change during split), so this
// header gives std::vector<hps::TreeNode> a deferred-free allocator: released blocks are kept intact in a
// small quarantine (the 64 most recent) before being returned to malloc, which makes the dangling read
// see the parent's unchanged values.  Nothing else about allocation changes.
#ifndef HPS_REF_COMPAT_HPP
#define HPS_REF_COMPAT_HPP

#include <cstddef>
#include <cstdlib>
#include <deque>
#include <memory>
#include <mutex>
#include <new>

namespace hps {
struct TreeNode;
}

namespace hps_ref_compat {
inline void quarantine_free(void* p) {
  static std::mutex mu;
  static std::deque<void*> q;
  std::lock_guard<std::mutex> lock(mu);
  q.push_back(p);
  while (q.size() > 64) {
    ::operator delete(q.front());
    q.pop_front();
  }
}
}  // namespace hps_ref_compat

template <>
struct std::allocator<hps::TreeNode> {
  using value_type = hps::TreeNode;
  using size_type = std::size_t;
  using difference_type = std::ptrdiff_t;
  using propagate_on_container_move_assignment = std::true_type;
  using is_always_equal = std::true_type;
  template <class U>
  struct rebind {
    using other = std::allocator<U>;
  };
  constexpr allocator() noexcept = default;
  template <class U>
  constexpr allocator(const std::allocator<U>&) noexcept {}
  hps::TreeNode* allocate(std::size_t n);
  void deallocate(hps::TreeNode* p, std::size_t) noexcept { hps_ref_compat::quarantine_free(p); }
  friend bool operator==(const allocator&, const allocator&) noexcept { return true; }
};

#include "hps/mesh.hpp"

inline hps::TreeNode* std::allocator<hps::TreeNode>::allocate(std::size_t n) {
  return static_cast<hps::TreeNode*>(::operator new(n * sizeof(hps::TreeNode)));
}

#endif
