// Defines the std::vector<double> overload of resample_sigma that the
// reference's stepper.cpp:313 calls but never declares or defines
// (SURVEY.md §0.2(a), Appendix A step 3).  The only possible semantics: run
// the SourceField overload (sources.cpp:66-75: zero sigma, then accumulate
// each spec's sigma over its rectangle in spec order) on the vector.
#include "swflood/stepper.hpp"

namespace swflood {

void resample_sigma(const std::vector<SourceSpec>& sources, double t,
                    const Terrain& terrain, std::vector<double>& sigma) {
  SourceField tmp;
  tmp.sigma.swap(sigma);
  resample_sigma(sources, t, terrain, tmp);
  tmp.sigma.swap(sigma);
}

}  // namespace swflood
